# A/B of environment settings (e.g. ZK_SMEM_KB=206): solve rate + per-phase times
for e in "$@"; do
  echo "== $e"
  env $e timeout 300 python bench.py --no-cpu --steps 3 --warmup 2 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=j['sub_metrics']['phases']
print(j['value'], j['sub_metrics']['bicgstab_iteration_us'], j['sub_metrics']['zspmv_us'], {k:p[k]['avg_us'] for k in ('spmv_t','spmv_pivot','true_res','setup')})"
done
