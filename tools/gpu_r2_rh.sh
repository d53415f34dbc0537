cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests/test_gpu_rhombus.py tests/test_gpu_errors.py tests/test_acceptance.py -m gpu -x -q --durations=15 > gpurun_out/pytest_rh.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_rh.log
timeout 300 python tools/rhombus_times.py > gpurun_out/rh_times.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/pytest_mr.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mr.log
