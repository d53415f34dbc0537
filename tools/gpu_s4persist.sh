# S4 persistent (2 CTAs per SM striding over units, tables staged once) vs one unit per CTA
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
HE_S4_PERSIST=2 timeout 900 python -m pytest tests/test_gpu_pcmm.py -x -q -k "llama_full_output or toy or spectral_equals" > gpurun_out/pytest_s4p.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_s4p.log
for v in 0 2 0 2; do
  export HE_S4_PERSIST=$v
  echo "$v $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']; print(d['value'], k['spectral_inverse'])")"
done > gpurun_out/s4p.txt 2>&1
