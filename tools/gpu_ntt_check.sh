# NTT users' GPU tests + the NTT bench
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_ringpack.py tests/test_gpu_rhombus.py tests/test_gpu_chain.py tests/test_gpu_slot_pcmm.py tests/test_gpu_stc.py -x -q > gpurun_out/pytest_nttc.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_nttc.log
timeout 300 python tools/bench_ntt.py 2>&1 | grep -v "^{" > gpurun_out/ntt_check.txt
