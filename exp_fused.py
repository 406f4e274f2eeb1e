import os, sys, json, subprocess
for env in ["", "SPOCK_FUSED_NOSTAGE=1 SPOCK_FUSED_OCC=4", "SPOCK_T_UNFUSED=1"]:
    cmd = (f"{env} python -c \"import sys, json; sys.path.insert(0,'.'); import bench; "
           f"print(json.dumps([bench.sweep_point(c, 1, 30, 6556.5) for c in ['c2','c2p','c3']]))\"")
    out = subprocess.run(cmd, shell=True, capture_output=True, text=True)
    print(env or "default", out.stdout.strip()[-1200:], out.stderr[-300:], flush=True)
