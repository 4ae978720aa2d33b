# Interleaved same-box A/B over several library builds: TAG CONFIG "SEEDS" LIB...
# ("" = the in-tree library; others are paths under tools/ab/)
out=gpurun_out/${1:-ab}_seeds.txt; cfg=$2; seeds=$3; shift 3
for rep in 1 2; do
for lib in "$@"; do
  if [ "$lib" = "-" ]; then v=""; else v="SC_LIB=$PWD/tools/ab/$lib"; fi
  echo "== $lib" >> $out
  env $v python tools/lcp_seeds.py $cfg --seeds $seeds >> $out 2>&1
done; done
python - "$out" <<'PY'
import json, sys
from collections import defaultdict
acc = defaultdict(list); lab = None
for l in open(sys.argv[1]):
    if l.startswith("=="): lab = l[3:].strip(); continue
    try: r = json.loads(l)
    except Exception: continue
    acc[lab].append((r["seed"], r["iters"], r["solve_ms"], r["us_per_iter"]))
for k, v in acc.items():
    print(f"{k:12s} us/iter {sum(x[3] for x in v)/len(v):6.2f}  mean solve {sum(x[2] for x in v)/len(v):6.2f} ms  iters {[x[1] for x in v[:len(v)//2]]}")
PY
