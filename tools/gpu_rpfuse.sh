cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_ringpack.py -x -q -k "fused or llama" -v > gpurun_out/pytest_rp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_rp.log
timeout 300 python tools/ringpack_times.py --method keyswitch1 > gpurun_out/ringpack_times_fused.txt 2>&1
HE_RP_UNFUSED=1 timeout 300 python tools/ringpack_times.py --method keyswitch1 > gpurun_out/ringpack_times_unfused.txt 2>&1
