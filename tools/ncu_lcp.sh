# true (non-event-inflated) durations of the LCP kernels, warm L2, for head vs new builds
for lib in head new; do
  for c in C4 C5; do
    if [ $lib = head ]; then export SC_LIB=$PWD/tools/ab/lib_head.so; else unset SC_LIB; fi
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:"gather|dt_kernel" -s 6 -c 6 --csv python tools/lcp_profile.py $c 10 2>/dev/null | grep -E '"(gpu__time|dram)' | python3 -c "
import sys,csv
for r in csv.reader(sys.stdin):
    print('$lib $c', r[4][:45], r[-3], r[-1])"
  done
done
