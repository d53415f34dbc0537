cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
export HE_S4_CLASSIC=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spec_inverse -s 1 -c 1 -o gpurun_out/s4_classic_l2 python tools/profile_op.py --ops 2 > gpurun_out/s4ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spec_gemm -s 2 -c 2 -o gpurun_out/s3_l2 python tools/profile_op.py --ops 2 >> gpurun_out/s4ncu.log 2>&1
