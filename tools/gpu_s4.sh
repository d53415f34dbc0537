cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in 0 1; do HE_SPEC_INV_SPLIT=$v timeout 900 python -m pytest tests/test_gpu_pcmm.py -x -q > gpurun_out/pytest_s4_$v.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_s4_$v.log; done
for v in 0 1 0 1; do echo "SPLIT=$v"; HE_SPEC_INV_SPLIT=$v timeout 300 python bench.py --no-direct --no-e2e --no-extras --cpu-rows 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels_ms'], d['roofline']['frac'])"; done > gpurun_out/bench_s4.txt 2>&1
