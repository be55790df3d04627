#!/bin/bash
# Time library variants (run under gpurun from the repo root):
#   VARIANTS="vA vB" CONFIGS="c5 c3" TESTS=1 tools/variants.sh
# Each build/<v>.so runs the GPU parity tests (TESTS=1) and short bench lines.
mkdir -p gpurun_out
for v in $VARIANTS; do
  export PASD_B200_LIB=$PWD/build/$v.so
  if [ "${TESTS:-0}" = 1 ]; then
    timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o timeout=120 > gpurun_out/t_$v.log 2>&1
    echo "$v tests rc=$? $(tail -1 gpurun_out/t_$v.log)"
  fi
  for c in ${CONFIGS:-c5 c3}; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_${v}_$c.json 2> gpurun_out/q_${v}_$c.err
    python - "$v" "$c" <<'PY'
import json, sys
v, c = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/q_{v}_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(v, c, "FAILED", e, open(f"gpurun_out/q_{v}_{c}.err").read()[-1500:]); sys.exit()
ms = d["ms_per_step"]; sh = d["roofline"]["kernel_time_shares"]
print(v, c, f"{ms:.3f} ms/it", {k: round(v * ms, 3) for k, v in sh.items() if v > 0.001}, "clk", d["clocks"]["sm_mhz"])
PY
  done
done
