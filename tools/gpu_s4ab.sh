# A/B of the S4 variants: PCMM parity tests with the default S4, then the op time with each variant
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pcmm.py -x -q > gpurun_out/pytest_s4ab.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_s4ab.log
for v in 1 1; do
  export HE_S4_PER_SM=$v
  echo "HE_S4_PER_SM=$v $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'], d['roofline']['frac'])")"
done > gpurun_out/bench_s4ab.txt 2>&1
