# r02d: A/B of library variants (pre-pass warps, forward diagonal probes) on the headline bench
T=r02d
mkdir -p gpurun_out
make -j8 all > gpurun_out/${T}_build.txt 2>&1
for v in "pre12 -DTTT_PRE_WARPS=12" "pre15 -DTTT_PRE_WARPS=15" "dnomath -DTTT_FWD_DIAG_MODE=1" "dnoload -DTTT_FWD_DIAG_MODE=2" "dpref -DTTT_FWD_DIAG_PREFETCH=1" "nofuse -DTTT_FWD_FUSED_DIAG=0"; do
  set -- $v; make variant VNAME=$1 EXTRA=$2 >> gpurun_out/${T}_build.txt 2>&1
done
bash bench_tools/ab_lib.sh $T 2 paper_2603_18567_b200/libtttattn.so build/libtttattn_pre12.so build/libtttattn_pre15.so build/libtttattn_dnomath.so build/libtttattn_dnoload.so build/libtttattn_dpref.so build/libtttattn_nofuse.so 2>&1 | tee gpurun_out/${T}_ab.txt
timeout 600 python -m pytest tests/test_gpu_bwd_unroll.py tests/test_gpu_check_mode.py tests/test_gpu_edge_cases.py -m gpu -q 2>&1 | tail -4
