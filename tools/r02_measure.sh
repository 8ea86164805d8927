#!/bin/bash
# Round-2 measurement session: the default bench line, a launch list of the
# bench command, and ncu --set full captures of the hot kernels per config
# (exported to CSV/text on the box: the .ncu-rep files are too large to bring back).
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python __graft_entry__.py smoke > gpurun_out/r02_smoke.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep --no-solvers > /dev/null 2>&1
K='regex:k_spmv2_phase_narrow|k_spmv_phase|k_s_update_pipe|k_xr_update_pipe|k_tt_ts_pass|k_pivot_pass|k_res_pass|k_p_next|k_zdot_pipe|k_znorm2_pipe|k_spmv'
for c in C4 C5 C3 C1; do
  ZK_PROFILE_CONFIG=$c timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 12 \
      -o /tmp/r02_prof_$c python tools/profile_kernels.py > gpurun_out/r02_prof_$c.log 2>&1
  ncu -i /tmp/r02_prof_$c.ncu-rep --page raw --csv > gpurun_out/r02_prof_${c}_raw.csv 2>/dev/null
  python tools/ncu_summary.py /tmp/r02_prof_$c.ncu-rep > gpurun_out/r02_ncu_summary_$c.txt 2>&1
done
ncu -i /tmp/r02_prof_C4.ncu-rep --page source --csv --kernel-name regex:k_xr_update_pipe --launch-skip 0 --launch-count 1 \
    > gpurun_out/r02_src_xr_update.csv 2>/dev/null
du -sh gpurun_out
