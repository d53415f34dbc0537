# S3 L2 policies: default (G normal, A last, C first) vs C normal / G first+C normal, interleaved
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in def 121 def 121 021 def; do
  if [ $v = def ]; then unset HE_S3_HINTS; else export HE_S3_HINTS=$v; fi
  echo "$v $(timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms']; print(d['value'], k['spectral_gemm_q0'], k['spectral_gemm_q1'], k['spectral_inverse'])")"
done > gpurun_out/s3hints2.txt 2>&1
