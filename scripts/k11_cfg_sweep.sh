#!/bin/bash
# K11 tile-configuration sweep at C3 (RPLU_K11_CFG 0/1/2), one bench line each.
mkdir -p gpurun_out/k11sweep
for c in ${CFGS:-0 1 2 3 4}; do
  RPLU_K11_CFG=$c timeout 600 python bench.py --config luerr --steps 3 --warmup 1 \
    > gpurun_out/k11sweep/cfg$c.log 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
line = json.loads(open(f"gpurun_out/k11sweep/cfg{c}.log").read().strip().splitlines()[-1])
r = line["roofline"]
print(f"cfg {c}: {r['achieved']:.2f} TFLOP/s frac {r['frac']:.3f} launch {r['avg_launch_ms']:.2f} ms "
      f"cublas {r['cublas_dgemm_tflops']:.2f} TF clocks {line['clocks']['sm_mhz']}")
PY
done
