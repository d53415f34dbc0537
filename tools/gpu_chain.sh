cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q > gpurun_out/pytest_chain.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_chain.log
python tools/chain_times.py 16 > gpurun_out/chain_times.txt 2>&1
