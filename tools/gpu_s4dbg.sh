cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in 0 2 3 6; do
  export HE_S4_WS_DBG=$v
  echo "DBG=$v $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['kernels_ms']['spectral_inverse'])")"
done > gpurun_out/bench_s4dbg.txt 2>&1
