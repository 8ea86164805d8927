#!/bin/bash
# A/B of env switches on one config's phases: tools/ab_env.sh <config> "<ENV=..>" ...
cfg=$1; shift
for spec in "$@"; do
  label=$(echo "$cfg $spec" | tr ' =' '__')
  env $spec python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu --no-sweep --no-solvers > gpurun_out/ab_$label.json 2>&1
done
