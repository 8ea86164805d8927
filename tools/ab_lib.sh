#!/bin/bash
# A/B of library builds on C4 phases: tools/ab_lib.sh <label>=<libzk.so path> ...
for spec in "$@"; do
  label=${spec%%=*}; lib=${spec#*=}
  ZK_LIB_PATH=$lib python bench.py --steps 3 --warmup 2 --no-cpu --no-sweep --no-solvers > gpurun_out/ab_$label.json 2>&1
done
