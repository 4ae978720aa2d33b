for cfg in C1 C2; do for env in 0 1; do
  SC_NO_PERSIST=$env timeout 300 python tools/bench_configs.py --configs $cfg --no-oracle 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg no_persist=$env', round(d['time_to_solution_ms'],3), 'ms iters', d['iters'], 'iters/s', round(d['bbpgd_iters_per_s']), d['kernel_launches'])"
done; done
