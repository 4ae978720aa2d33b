out=gpurun_out/${1:-ab}_batch.txt
for rep in 1 2; do
for b in "" "SC_BATCH=16" "SC_BATCH=32" "SC_BATCH=64"; do
  echo "== $b" >> $out
  env $b python tools/lcp_time.py C4 C2 >> $out 2>&1
done; done
python examples/piston.py 4096 40 > gpurun_out/${1:-ab}_piston.txt 2>&1
