# Interleaved same-box A/B of the C4 LCP loop: the in-tree library vs tools/ab/lib_prev.so
# (usage: bash tools/ab/ab_c4.sh TAG [REPS])
out=gpurun_out/${1:-ab}_lcp.txt
AB=$PWD/tools/ab
for rep in $(seq 1 ${2:-3}); do
for v in "" "SC_LIB=$AB/lib_prev.so"; do
  echo "== $v" >> $out
  env $v python tools/lcp_time.py C4 >> $out 2>&1
done; done
