#!/bin/bash
# A/B of library builds on one config's phases (CFG, default C4): tools/ab_lib.sh <label>=<libzk.so path> ...
cfg=${CFG:-C4}
for spec in "$@"; do
  label=${spec%%=*}; lib=${spec#*=}
  ZK_LIB_PATH=$lib python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu --no-sweep --no-solvers > gpurun_out/ab_${cfg}_$label.json 2>&1
done
