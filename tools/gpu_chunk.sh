cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for cfg in "0 120" "256 120" "256 121" "256 122" "512 121" "512 122"; do
  set -- $cfg
  export HE_SPEC_CHUNK=$1 HE_S3_HINTS=$2
  echo "CHUNK=$1 HINTS=$2 $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'], d['parity']['words_equal'] if 'parity' in d else '')")"
done > gpurun_out/bench_chunk.txt 2>&1
