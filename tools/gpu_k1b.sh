cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for bn in 0 32 0 32; do
  export HE_GEMM_BN=$bn
  echo "BN=$bn $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'])")"
done > gpurun_out/bench_k1b.txt 2>&1
