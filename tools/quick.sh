#!/bin/bash
# Quick GPU check (run under gpurun from the repo root): GPU parity tests, then
# short C5 / C3 bench lines reduced to the numbers that move.
#   tools/quick.sh [pytest-args]
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -o timeout=120 "$@" > gpurun_out/t.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/t.log)"
for c in ${QUICK_CONFIGS:-c5 c3}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/q_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", e, open(f"gpurun_out/q_{c}.err").read()[-2000:]); sys.exit()
ms = d["ms_per_step"]; sh = d["roofline"]["kernel_time_shares"]
print(c, f"{ms:.3f} ms/it", {k: round(v * ms, 3) for k, v in sh.items() if v > 0.001}, "frac", d["roofline"]["frac"], "clk", d["clocks"]["sm_mhz"])
PY
done
