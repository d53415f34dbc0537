cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q -s > gpurun_out/pytest_cts.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_cts.log
