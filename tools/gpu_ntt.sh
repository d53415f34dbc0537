cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_ntt.py -x -q > gpurun_out/pytest_ntt.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ntt.log
for cfg in 4 6 7 4; do echo "MINB $cfg"; HE_NTT_MINB=$cfg timeout 300 python tools/bench_ntt.py | grep -v "^{" | grep limb=0; done > gpurun_out/bench_ntt.txt 2>&1
