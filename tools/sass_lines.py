"""Per-source-line instruction and stall-sample totals of one kernel from an
ncu report: ncu's SASS source page (per-instruction "Instructions Executed"
and warp-stall samples) joined with nvdisasm -g line info of the same cubin.
Usage: python tools/sass_lines.py <sass.csv> <nvdisasm -g output> <kernel symbol substring> [top]
(sass.csv: ncu -i rep --page source --csv --print-source sass)."""
import collections
import csv
import re
import sys


def main():
    sass, dis, sym = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(sass)))
    hdr = rows[1]
    ie, ss, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    data = [r for r in rows[2:] if r and r[ie].isdigit()]
    base = int(data[0][0], 16)
    # offset -> (file, line) from nvdisasm -g of the matching function section
    lines = {}
    cur = None
    insec = False
    for ln in open(dis):
        if ln.startswith(".text."):
            insec = sym in ln
            continue
        if not insec:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            lines[int(m.group(1), 16)] = cur
    agg_i, agg_s = collections.Counter(), collections.Counter()
    tot_i = tot_s = 0
    for r in data:
        off = int(r[0], 16) - base
        key = lines.get(off, ("?", 0))
        agg_i[key] += int(r[ie])
        agg_s[key] += int(r[ss])
        tot_i += int(r[ie])
        tot_s += int(r[ss])
    print(f"instructions {tot_i}, stall samples {tot_s}, mapped offsets {len(lines)}")
    for key, s in agg_s.most_common(top):
        print(f"{key[0]}:{key[1]:5d}  samples {100.0 * s / tot_s:5.1f}%  inst {100.0 * agg_i[key] / tot_i:5.1f}%")


if __name__ == "__main__":
    main()
