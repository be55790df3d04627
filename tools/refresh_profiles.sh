#!/bin/bash
# Round evidence on a B200 (run under gpurun from the repo root):
#   tools/refresh_profiles.sh r02
# Writes gpurun_out/prof/<round>_*: bench lines for C1-C5 (+ the fp32 mode at C5) and the
# reference arm, the C1 whole-solve comparison, the ncu launch list of a short C5 run and one
# `ncu --set full` capture of an iteration's kernels.  Copy the ones to keep into profiles/.
set -u
R=${1:-r02}
O=gpurun_out/prof
mkdir -p $O
python bench.py --steps 20 --warmup 3 > $O/${R}_bench_c5.json 2> $O/${R}_bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/${R}_bench_reference_c5.json 2> $O/${R}_bench_reference_c5.err
python tools/c1_solve.py > $O/${R}_c1_solve.json 2> $O/${R}_c1_solve.err
for c in c1 c2 c3 c4; do
  python bench.py --config $c --steps 20 --warmup 3 > $O/${R}_bench_$c.json 2> $O/${R}_bench_$c.err
done
python bench.py --dtype f32 --steps 10 --warmup 3 --no-cpu-baseline > $O/${R}_bench_c5_f32.json 2> $O/${R}_bench_c5_f32.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --steady-after 0 --profile-iters 1"
$CMD > $O/ncu_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 60 --csv \
  --log-file $O/${R}_launches_c5.csv $CMD > $O/ncu_launch.log 2>&1
$CMD > $O/ncu_plain2.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:'^k_' --launch-skip 20 --launch-count 11 \
  -o $O/${R}_c5_full $CMD > $O/ncu_full.log 2>&1
ls -la $O
