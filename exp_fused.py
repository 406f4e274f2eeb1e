import os, sys, json, subprocess
cfgs = sys.argv[1] if len(sys.argv) > 1 else "c2,c2p,c3"
envs = ["", "SPOCK_FUSED_FT=256 SPOCK_FUSED_SLOTS=2 SPOCK_FUSED_STAGEALL=1",
        "SPOCK_FUSED_FT=128 SPOCK_FUSED_SLOTS=1 SPOCK_FUSED_STAGEALL=1",
        "SPOCK_FUSED_FT=128 SPOCK_FUSED_SLOTS=2 SPOCK_FUSED_STAGEALL=0",
        "SPOCK_FUSED_FT=256 SPOCK_FUSED_SLOTS=1 SPOCK_FUSED_STAGEALL=0",
        "SPOCK_FUSED_FT=128 SPOCK_FUSED_SLOTS=1 SPOCK_FUSED_STAGEALL=0 SPOCK_FUSED_NOSTAGE=1"]
for env in envs:
    cmd = (f"{env} python -c \"import sys, json; sys.path.insert(0,'.'); import bench; "
           f"print(json.dumps([(lambda d: (d['config'], round(d['ms_per_T'],4), round(d['T_frac'],3)))(bench.sweep_point(c, 1, 30, 6556.5)) for c in '{cfgs}'.split(',')]))\"")
    out = subprocess.run(cmd, shell=True, capture_output=True, text=True)
    print(env or "auto", out.stdout.strip()[-600:], out.stderr[-300:], flush=True)
