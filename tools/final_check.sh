#!/bin/bash
# Round-end check on the GPU box: sanitizers on the fused T and the cluster loop, smoke(), pytest -m gpu,
# bench.py and its reference arm (outputs under gpurun_out/).  Usage: bash tools/final_check.sh
cd "$GRAFT_REPO_ROOT"
run() { local name=$1 envs=$2 tool=$3; shift 3; local out; out=$(env $envs timeout -s KILL 900 compute-sanitizer --tool "$tool" --print-limit 5 "$@" 2>&1); echo "$name [$tool] $(echo "$out" | grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' | tail -1) $(echo "$out" | grep -o 'ok [a-z]*' | tail -1)"; echo "$out" | grep -E "Error|Thread \(" | sort | uniq -c | head -6; }
for tool in racecheck memcheck synccheck; do
  run "T fused (register GEMVs)" "" $tool python tools/few_T.py c2
  run "solve cluster-resident loop (c1, 8 CTAs)" "SPOCK_CLUSTER=1" $tool python tools/solve_kernels.py c1 6 solve
done > gpurun_out/sanitize_final4.txt 2>&1
cat gpurun_out/sanitize_final4.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final4.log 2>&1; tail -2 gpurun_out/smoke_final4.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final4.txt 2>&1; tail -3 gpurun_out/pytest_gpu_final4.txt
timeout 900 python bench.py > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err; tail -c 200 gpurun_out/bench_final4.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_final4_ref.json 2>gpurun_out/bench_final4_ref.err; tail -c 200 gpurun_out/bench_final4_ref.json
