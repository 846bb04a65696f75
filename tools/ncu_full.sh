#!/bin/bash
# ncu --set full captures of steady-state launches of the top kernels of one
# bench step (python bench.py --ncu). Usage: tools/ncu_full.sh "regex:skip:count" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "$@"; do
  pat=${spec%%:*}; rest=${spec#*:}; skip=${rest%%:*}; cnt=${rest##*:}
  tag=$(echo "$pat" | tr -c 'A-Za-z0-9_' '_' | cut -c1-40)
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$pat" -s $skip -c $cnt \
    -o gpurun_out/full_$tag -f python bench.py --ncu > gpurun_out/full_$tag.log 2>&1
  echo "ncu full $pat exit $?"
done
