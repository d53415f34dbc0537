# K1 knob sweep: tile width, raster group, L2 hints (timing + DRAM bytes per launch)
cd $GRAFT_REPO_ROOT
./tools/tma_overlap_probe > gpurun_out/tma_probe.txt 2>&1
run() {  # label env...
  label=$1; shift
  t=$(env "$@" timeout 120 python tools/gpu_check.py --time 2>&1 | grep "^shape" | sed 's/.*gemm \([0-9.]*\) ms.*/\1/')
  b=$(env "$@" timeout 200 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:modgemm -s 1 -c 1 --csv python tools/profile_op.py 2>/dev/null | grep -E "dram__bytes_read|tensor_cycles" | awk -F'","' '{print $(NF-2)" "$(NF-1)" "$NF}' | tr '\n' ' ')
  echo "$label | gemm_ms=$t | $b" >> gpurun_out/sweep.txt
}
run default
run bn32 HE_GEMM_BN=32
run gm1 HE_GEMM_GROUP_M=1
run gm2 HE_GEMM_GROUP_M=2
run gm4 HE_GEMM_GROUP_M=4
run gm16 HE_GEMM_GROUP_M=16
run bnormal HE_GEMM_HINT_B=normal
run gm4_bnormal HE_GEMM_GROUP_M=4 HE_GEMM_HINT_B=normal
run anormal_bnormal HE_GEMM_HINT_A=normal HE_GEMM_HINT_B=normal
cat gpurun_out/tma_probe.txt gpurun_out/sweep.txt
