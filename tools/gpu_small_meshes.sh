#!/bin/bash
# Throughput and K1/K2 shares on reduced C5 meshes (launch-overhead check).
mkdir -p gpurun_out
for b in 80 160 320; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --base-n $b > gpurun_out/small_$b.log 2>&1
  python - "$b" <<'PY'
import json, sys
b = sys.argv[1]
d = json.loads(open(f"gpurun_out/small_{b}.log").read().strip().splitlines()[-1])
r = d["roofline"]
print(b, d["config"]["K_per_rank"], "%.3e" % d["value"], round(d["ms_per_step"], 3), round(r["k1_share_of_step"], 3),
      round(r["k2_share_of_step"], 3))
PY
done
