# A/B: S4 with compile-time moduli (immediate q operands) vs the moduli as kernel parameters
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pcmm.py -x -q > gpurun_out/pytest_s4kq.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_s4kq.log
for v in kq rt kq rt; do
  if [ $v = rt ]; then export HE_S4_RUNTIME_Q=1; else unset HE_S4_RUNTIME_Q; fi
  echo "$v $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'], d['roofline']['frac'])")"
done > gpurun_out/bench_s4kq.txt 2>&1
