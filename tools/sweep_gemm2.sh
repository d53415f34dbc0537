cd $GRAFT_REPO_ROOT
run() {  # label env...
  label=$1; shift
  t=$(env "$@" timeout 120 python tools/gpu_check.py --time 2>&1 | grep "^shape" | sed 's/.*gemm \([0-9.]*\) ms.*all \(.*\)/\1 \2/')
  b=$(env "$@" timeout 200 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:modgemm -s 1 -c 1 --csv python tools/profile_op.py 2>/dev/null | grep -E "dram__bytes_read|tensor_cycles|duration" | awk -F'","' '{print $(NF-2)" "$(NF-1)" "$NF}' | tr '\n' ' ')
  echo "$label | gemm_ms=$t | $b" >> gpurun_out/sweep2.txt
}
run default
run pairs72 HE_GEMM_PAIRS=72
run pairs72_gm16 HE_GEMM_PAIRS=72 HE_GEMM_GROUP_M=16
run gm16 HE_GEMM_GROUP_M=16
run pairs64_gm16 HE_GEMM_PAIRS=64 HE_GEMM_GROUP_M=16
cat gpurun_out/sweep2.txt
