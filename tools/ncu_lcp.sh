# true durations of the LCP kernels (warm L2): committed build (SC_LIB=tools/ab/lib_head.so) vs working tree
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
  prof head $c SC_LIB=$PWD/tools/ab/lib_head.so
  prof new $c
done
