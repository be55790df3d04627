#!/bin/bash
# FP64 roofline denominator with the SM clocks recorded while it runs
# (run under gpurun from the repo root):  tools/fp64_peak.sh > profiles/rNN_fp64_peak.txt
set -u
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
nvidia-smi --id=0 --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active \
  --format=csv,noheader -lms 200 > /tmp/fp64_clocks.csv &
SMI=$!
sleep 0.5
tools/fp64_peak 5
kill $SMI
python3 - <<'PY'
import statistics
rows = [l.strip().split(", ") for l in open("/tmp/fp64_clocks.csv") if l.strip()]
sm = [float(r[1].split()[0]) for r in rows]
mx = [float(r[2].split()[0]) for r in rows]
pw = [float(r[3].split()[0]) for r in rows if r[3].split()[0].replace('.', '').isdigit()]
reasons = sorted(set(r[5] for r in rows))
print('{"clocks": {"samples": %d, "sm_mhz_median": %s, "sm_mhz_min": %s, "sm_max_mhz": %s, "power_w_max": %s, "event_reasons_active": %s}}'
      % (len(sm), statistics.median(sm), min(sm), max(mx), max(pw) if pw else None, '["' + '", "'.join(reasons) + '"]'))
PY
