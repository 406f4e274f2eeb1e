"""Command-line front end (SPEC.md module cli): generation, profile emission on
CPU; solve and bench verbs on the GPU."""
import csv
import math
import os
import subprocess
import sys

import pytest

from paper_2505_12078_b200.__main__ import main, performance_profile
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.problem_io import load_problem, save_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_generate_random_desk_scale_is_deterministic(tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    assert main(["generate-random", "--seed", "3", "--count", "2", "--out", str(a), "--desk-scale"]) == 0
    assert main(["generate-random", "--seed", "3", "--count", "2", "--out", str(b), "--desk-scale"]) == 0
    names = sorted(os.listdir(a))
    assert names == ["case1_seed3.spk", "case1_seed4.spk"]
    for n in names:
        assert (a / n).read_bytes() == (b / n).read_bytes()
        p = load_problem(str(a / n))
        nv = p.nx * p.tree.num_nodes() + p.nu * p.tree.num_nonleaf()
        assert 1000 <= nv <= 10000 and p.nx == 2 * p.nu  # SPEC.md cli gen_random_suite, desk scale


def test_performance_profile():
    rows = [{"problem": "p1", "solver": "spock", "wall_s": "1.0", "reason": "converged"},
            {"problem": "p1", "solver": "cp", "wall_s": "2.0", "reason": "converged"},
            {"problem": "p2", "solver": "spock", "wall_s": "5.0", "reason": "max_iters"},
            {"problem": "p2", "solver": "cp", "wall_s": "3.0", "reason": "converged"}]
    prof = performance_profile(rows)
    f = {(r["solver"], r["tau"]): r["fraction_solved"] for r in prof}
    assert f[("spock", 1.0)] == 0.5 and f[("cp", 1.0)] == 0.5
    assert f[("cp", 2.0)] == 1.0 and f[("spock", 2.0)] == 0.5  # spock's failure has ratio inf


def test_profile_emit(tmp_path):
    src = tmp_path / "bench.csv"
    with open(src, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=["problem", "solver", "wall_s", "reason"])
        w.writeheader()
        w.writerow({"problem": "p", "solver": "cp", "wall_s": "1", "reason": "converged"})
    out = tmp_path / "prof.csv"
    assert main(["profile-emit", str(src), "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert rows[0]["solver"] == "cp" and float(rows[0]["fraction_solved"]) == 1.0


@pytest.mark.gpu
def test_solve_verb_exit_codes(tmp_path):
    p = make_config("c1", seed=1)
    f = tmp_path / "c1.spk"
    save_problem(str(f), p)
    cmd = [sys.executable, "-m", "paper_2505_12078_b200", "solve", str(f), "--algorithm", "cp",
           "--out", str(tmp_path / "sol.spk")]
    ok = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    assert ok.returncode == 0, ok.stderr[-500:]  # CP converges on c1 (41 689 iterations)
    assert (tmp_path / "sol.spk").exists()
    bad = subprocess.run(cmd[:-2] + ["--max-iters", "1"], cwd=ROOT, capture_output=True, text=True)
    assert bad.returncode == 1 and '"reason": "max_iters"' in bad.stdout


@pytest.mark.gpu
def test_bench_verb(tmp_path):
    d = tmp_path / "suite"
    assert main(["generate-random", "--seed", "1", "--count", "2", "--out", str(d), "--desk-scale"]) == 0
    out, prof = tmp_path / "b.csv", tmp_path / "p.csv"
    assert main(["bench", str(d), "--out", str(out), "--profile-out", str(prof), "--max-iters", "50",
                 "--time-limit-s", "60"]) == 0
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 4 and {r["solver"] for r in rows} == {"spock", "cp"}
    assert all(int(r["n_v"]) >= 1000 for r in rows)
    assert list(csv.DictReader(open(prof)))
