cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in 0 1; do
  if [ $v = 1 ]; then export HE_S4_V1=1; else unset HE_S4_V1; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:spec_inverse -s 1 -c 1 -o gpurun_out/s4_v$v python tools/profile_op.py --ops 2 > gpurun_out/s4ncu_v$v.log 2>&1
done
unset HE_S4_V1
timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'], d['roofline']['frac'])" > gpurun_out/bench_s4v2b.txt 2>&1
