cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_ntt.py -m gpu -x -q > gpurun_out/pytest_ntt.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ntt.log
timeout 300 python tools/bench_ntt.py > gpurun_out/bench_ntt.txt 2>&1
HE_NTT_NO_PERSIST=1 timeout 300 python tools/bench_ntt.py > gpurun_out/bench_ntt_twopass.txt 2>&1
timeout 300 python tools/ringpack_times.py > gpurun_out/ringpack_times.txt 2>&1
