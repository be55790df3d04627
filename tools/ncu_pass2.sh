set -e
CMD="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --steady-after 0 --profile-iters 1"
for v in base probe3; do
  PASD_B200_LIB=$PWD/build/$v.so $CMD > gpurun_out/plain_$v.log 2>&1
  PASD_B200_LIB=$PWD/build/$v.so ncu --set full --clock-control none --import-source on -k regex:k_pass2_fused -s 2 -c 1 -o gpurun_out/p2_$v $CMD > gpurun_out/ncu_$v.log 2>&1
done
