# Time to solution over seeds, in-tree library vs tools/ab/lib_prev.so (usage: TAG CONFIG SEEDS...)
out=gpurun_out/${1:-ab}_seeds.txt; cfg=${2:-C4}; shift 2
AB=$PWD/tools/ab
for v in "" "SC_LIB=$AB/lib_prev.so" "" "SC_LIB=$AB/lib_prev.so"; do
  echo "== $v" >> $out
  env $v python tools/lcp_seeds.py $cfg --seeds "$@" >> $out 2>&1
done
