out=gpurun_out/${1:-ab}_lcp.txt
AB=$PWD/tools/ab
for rep in 1 2; do
for v in "" "SC_LIB=$AB/lib_notrig.so" "SC_LIB=$AB/lib_nowait.so" "SC_LIB=$AB/lib_prev.so"; do
  echo "== $v" >> $out
  env $v python tools/lcp_time.py C4 >> $out 2>&1
done; done
