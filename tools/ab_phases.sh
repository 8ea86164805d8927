# A/B of libzk variants under exp/<name>/libzk.so: solve rate + per-phase times
for d in "$@"; do
  echo "== $d"
  ZK_LIB_PATH=exp/$d/libzk.so timeout 300 python bench.py --no-cpu --steps 3 --warmup 2 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=j['sub_metrics']['phases']
print(j['value'], j['sub_metrics']['bicgstab_iteration_us'], {k:p[k]['avg_us'] for k in ('s_update','xr_update','spmv_t','spmv_pivot','true_res','p_next')})"
done
