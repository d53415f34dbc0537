cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
HE_S4_GTW=1 timeout 900 python -m pytest tests/test_gpu_pcmm.py -x -q > gpurun_out/pytest_gtw.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gtw.log
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export HE_S4_GTW=1; else unset HE_S4_GTW; fi
  echo "GTW=$v $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'])")"
done > gpurun_out/bench_gtw.txt 2>&1
