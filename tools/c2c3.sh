for c in C2 C3; do
  timeout 300 python tools/bench_configs.py --configs $c --no-oracle 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['kernel_launches']
print('$c', round(d['time_to_solution_ms'],2), 'rpy ms/launch', round(k['rpy']/n['rpy'],4), 'frac', round(d['rpy_frac_fp64_peak'],3), 'iters', d['iters'])"
done
