# true (non-event-inflated) durations of the LCP kernels, warm L2: single-list vs split D-gather
prof() {  # label, config, env...
  env "${@:3}" ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none \
      -k regex:"gather|dt_kernel" -s 6 -c 6 --csv python tools/lcp_profile.py $2 10 2>/dev/null \
    | grep -E '"gpu__time' | python3 -c "
import sys,csv,collections
d=collections.defaultdict(list)
for r in csv.reader(sys.stdin):
    d[r[4].split('(')[0].split('::')[-1][:40]].append(float(r[-1]))
print('$1 $2', {k: round(sum(v)/len(v)/1000,2) for k,v in d.items()})"
}
for c in C4 C5; do
  prof single $c SC_NO_GATHER_SPLIT=1
  prof split $c
done
