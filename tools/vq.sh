#!/bin/bash
# Quick A/B of library variants (run under gpurun from the repo root): pass-2 parity tests + short bench lines.
#   VARIANTS="a b" CONFIGS="c5 c3" tools/vq.sh        ("default" = the in-tree library)
mkdir -p gpurun_out
for v in $VARIANTS; do
  if [ "$v" = default ]; then unset PASD_B200_LIB; else export PASD_B200_LIB=$PWD/build/$v.so; fi
  [ "${SKIP_TESTS:-0}" = 1 ] || timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "single_step or trivial_phase or steady_state" > gpurun_out/vq_$v.log 2>&1
  echo "$v tests rc=$? $(tail -1 gpurun_out/vq_$v.log)"
  for c in ${CONFIGS:-c5}; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --steady-after 0 > gpurun_out/vq_${v}_$c.json 2> gpurun_out/vq_${v}_$c.err
    python - "$v" "$c" <<'PY'
import json, sys
v, c = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/vq_{v}_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(v, c, "FAILED", e, open(f"gpurun_out/vq_{v}_{c}.err").read()[-1500:]); sys.exit()
ms = d["ms_per_step"]; r = d["roofline"]
print(v, c, f"{ms:.3f} ms/it", {k: round(x["ms_per_launch"], 3) for k, x in r["per_kernel"].items()}, "clk", d["clocks"]["sm_mhz"])
PY
  done
done
