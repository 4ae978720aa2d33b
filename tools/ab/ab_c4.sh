out=gpurun_out/${1:-ab}_lcp.txt
for rep in 1 2 3; do
for v in "" "SC_NO_GRAPHS=1"; do
  echo "== $v" >> $out
  env $v python tools/lcp_time.py C4 C2 >> $out 2>&1
done; done
