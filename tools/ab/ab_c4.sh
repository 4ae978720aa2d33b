out=gpurun_out/${1:-ab}_lcp.txt
AB=$PWD/tools/ab
for rep in 1 2 3; do
for lib in "" "SC_LIB=$AB/lib_prev.so"; do
  echo "== $lib" >> $out
  env $lib python tools/lcp_time.py C4 >> $out 2>&1
done; done
