#!/bin/bash
# Steady-state (full-rank phase) iteration times: per config, warm up W
# iterations into the full-rank phase, then time 20 (run under gpurun).
#   STEADY="c3:150 c4:150 c5:130" tools/steady.sh
for cw in ${STEADY:-c3:150 c4:150 c5:130}; do
  c=${cw%%:*}; w=${cw##*:}
  timeout 600 python bench.py --config $c --steps 20 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/st_$c.json 2> gpurun_out/st_$c.err
  python - "$c" "$w" <<'PY'
import json, sys
c, w = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/st_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", e); sys.exit()
ms = d["ms_per_step"]
print(c, f"after {w}: {ms:.3f} ms/it", {k: round(v * ms, 3) for k, v in d["roofline"]["kernel_time_shares"].items() if v > 0.001})
PY
done
