#!/bin/bash
# A/B of BiCGStab loop shapes on C4 (env switches in zk_bicgstab.cu make_launch)
for cfg in "ZK_RESPASS=0" "ZK_RESPASS=1"; do
  env $cfg python bench.py --steps 3 --warmup 2 --no-cpu --no-sweep --no-solvers > gpurun_out/ab_$(echo $cfg | tr ' =' '__').json 2>&1
done
