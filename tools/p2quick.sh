#!/bin/bash
# Pass-2 iteration loop (run under gpurun): pass-2 parity tests, then C5 / C3
# lines reduced to the per-kernel split.   tools/p2quick.sh [tag]
T=${1:-x}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "single_step or trivial_phase or steady_state" > gpurun_out/p2q_$T.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/p2q_$T.log)"
for c in ${QUICK_CONFIGS:-c5 c3}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --steady-after 0 > gpurun_out/p2q_${T}_$c.json 2> gpurun_out/p2q_${T}_$c.err
  python - "$c" "$T" <<'PY'
import json, sys
c, t = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/p2q_{t}_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", e, open(f"gpurun_out/p2q_{t}_{c}.err").read()[-2000:]); sys.exit()
ms = d["ms_per_step"]; r = d["roofline"]
print(c, f"{ms:.3f} ms/it", {k: v["ms_per_launch"] for k, v in r["per_kernel"].items()}, "frac", r["frac"], "clk", d["clocks"]["sm_mhz"])
PY
done
