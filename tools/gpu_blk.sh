cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_pcmm.py -x -q -k "last_row_block" --durations=10 > gpurun_out/pytest_blk.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_blk.log
