#!/bin/bash
# compute-sanitizer sweep over every T schedule and the solve loop (GPU box):
#   bash tools/sanitize.sh > gpurun_out/sanitize.txt
# racecheck (shared-memory hazards), synccheck (barrier misuse) and memcheck (out-of-bounds / misaligned
# global and shared accesses) on c2 (223 nodes) -- the device-side setup kernels run in every
# solver construction -- and the cluster-resident loop on c1; prints one summary per run.
cd "$(dirname "$0")/.."
run() {  # name, env, tool, command...
  local name=$1 envs=$2 tool=$3; shift 3
  local out
  out=$(env $envs timeout -s KILL 900 compute-sanitizer --tool "$tool" --print-limit 5 "$@" 2>&1)
  echo "$name [$tool] $(echo "$out" | grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' | tail -1) $(echo "$out" | grep -o 'ok [a-z]*' | tail -1)"
  echo "$out" | grep -E "Error|Thread \(" | sort | uniq -c | head -6
}
for tool in racecheck memcheck synccheck; do
  run "T fused" "" $tool python tools/few_T.py c2
  run "T wide" "SPOCK_T_UNFUSED=1 SPOCK_T_WIDE=1" $tool python tools/few_T.py c2
  run "T stages" "SPOCK_T_UNFUSED=1 SPOCK_T_WIDE=0" $tool python tools/few_T.py c2
  run "solve host loop (L, L*, reductions, loop kernels)" "SPOCK_SOLVE_GRAPH=0" $tool python tools/solve_kernels.py c2 4 solve
  run "solve cluster-resident loop (c1)" "SPOCK_CLUSTER=1" $tool python tools/solve_kernels.py c1 6 solve
done
