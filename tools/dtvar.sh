# A/B of LCP-kernel variants: per-launch gather / D^T times (C4 rods, C5 spheres)
run() {  # config, label, env...
  env "${@:3}" timeout 300 python tools/bench_configs.py --configs $1 --no-oracle 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms']; n=d['kernel_launches']
print('$1 $2', round(d['time_to_solution_ms'],2), 'gather us', round(1000*k['gather']/n['gather'],2), 'dt us', round(1000*k['dt']/n['dt'],2), 'iters', d['iters'], 'res', d['residual'])"
}
for c in C4 C5; do
run $c head SC_LIB=$PWD/tools/ab/lib_head.so
run $c new
done
