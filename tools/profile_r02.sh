# round-2 profiles: launch list of one bench step, one --set full capture of the symmetric RPY
# kernel (bench configuration, C5) and of the C4 LCP kernels (a3 gather, a5 D^T).  One ncu use per
# gpurun call; every command ran plain (exit 0) right before its ncu run.
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$B > gpurun_out/p02_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/p02_launches.csv \
    $B > gpurun_out/p02_ncu_launch.log 2>&1
$B > gpurun_out/p02_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rpy_sym_kernel -s 3 -c 1 -o gpurun_out/p02_rpy_sym \
    $B > gpurun_out/p02_ncu_full.log 2>&1
# (SC_NO_GRAPHS=1: ncu cannot profile the kernel nodes of a graph with a conditional node)
SC_NO_GRAPHS=1 python tools/lcp_profile.py C4 10 > gpurun_out/p02_plain3.log 2>&1 && \
SC_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel|dt_kernel" -s 8 -c 4 \
    -o gpurun_out/p02_lcp_c4 python tools/lcp_profile.py C4 10 > gpurun_out/p02_ncu_lcp.log 2>&1
python tools/fmm_scaling.py --min-log2n 20 --max-log2n 20 --direct-max-log2n 0 --orders 6 > gpurun_out/p02_plain4.log 2>&1 && \
ncu --set full --clock-control none -k regex:"m2l_kernel|l2p_p2p_kernel" -c 2 -o gpurun_out/p02_fmm \
    python tools/fmm_scaling.py --min-log2n 20 --max-log2n 20 --direct-max-log2n 0 --orders 6 > gpurun_out/p02_ncu_fmm.log 2>&1
ls -la gpurun_out/ | grep p02
