#!/bin/bash
# tools/steady.sh for each build/<v>.so in $VARIANTS (plus GPU tests when TESTS=1)
for v in $VARIANTS; do
  export PASD_B200_LIB=$PWD/build/$v.so
  if [ "${TESTS:-0}" = 1 ]; then
    timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o timeout=200 -k "not client_matches" > gpurun_out/t_$v.log 2>&1
    echo "$v tests rc=$? $(tail -1 gpurun_out/t_$v.log)"
  fi
  tools/steady.sh | sed "s/^/$v /"
done
