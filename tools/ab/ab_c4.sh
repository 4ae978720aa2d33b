# interleaved same-box A/B of the C4 (rods) LCP loop variants; tools/lcp_time.py per variant
out=gpurun_out/${1:-ab}_lcp.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_walls.py -k "rods or C4 or moving" -q -p no:cacheprovider -x > gpurun_out/${1:-ab}_tests.log 2>&1
tail -3 gpurun_out/${1:-ab}_tests.log >> $out
for rep in 1 2; do
for p in "" "SC_RODS_INC=0 SC_NO_PERSIST=1" "SC_RODS_INC=0 SC_LCP_VARIANT=2" "SC_NO_GRAPHS=1"; do
  echo "== $p" >> $out
  env $p python tools/lcp_time.py C4 >> $out 2>&1
done; done
