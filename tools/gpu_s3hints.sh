cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1

for h in 120 121 122 220 110; do
  export HE_S3_HINTS=$h
  echo "HINTS=$h $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'])")"
done > gpurun_out/bench_s3hints.txt 2>&1
