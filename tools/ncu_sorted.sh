for c in C4 C5; do for o in random sorted; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none \
      -k regex:"gather|dt_kernel" -s 6 -c 6 --csv python tools/lcp_sorted_probe.py $c $o 10 2>/dev/null \
    | grep -E '"(gpu__time|dram)' | python3 -c "
import sys,csv,collections
d=collections.defaultdict(list)
for r in csv.reader(sys.stdin):
    d[(r[4].split('(')[0].split('::')[-1][:30], r[-3][:12])].append(float(r[-1]))
print('$c $o', {k: round(sum(v)/len(v)/ (1000 if 'time' in k[1] else 1e6),2) for k,v in d.items()})"
done; done
