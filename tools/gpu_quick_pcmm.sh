# PCMM GPU tests + the headline bench line (no side blocks) for a quick check of a K7 change
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pcmm.py -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_quick.log
for i in 1 2; do
  timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels_ms'], d['roofline']['frac'])"
done > gpurun_out/bench_quick.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ringpack.py -x -q > gpurun_out/pytest_quick_rp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_quick_rp.log
