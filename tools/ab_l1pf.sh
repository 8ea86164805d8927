for d in pf0 pf1 pf2 pf3; do
  echo "== $d"
  ZK_LIB_PATH=exp/$d/libzk.so timeout 120 python tools/l1_timing.py 2>&1 | tail -1
  ZK_LIB_PATH=exp/$d/libzk.so timeout 300 python bench.py --no-cpu --steps 2 --warmup 1 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=j['sub_metrics']['phases']
print(j['value'], j['sub_metrics']['bicgstab_iteration_us'], {k:p[k]['avg_us'] for k in ('s_update','xr_update','spmv_t','spmv_pivot','true_res','p_next')})"
done
