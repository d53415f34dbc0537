# ring packing: rows-pass final reduction moved into the MAC (default) vs HE_RP_NTT_REDUCE=1
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_ringpack.py tests/test_gpu_ntt.py -x -q > gpurun_out/pytest_rplazy.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_rplazy.log
for v in lazy lazy; do
  if [ $v = reduce ]; then export HE_RP_NTT_REDUCE=1; else unset HE_RP_NTT_REDUCE; fi
  echo "== $v" >> gpurun_out/rplazy.txt
  timeout 300 python tools/ringpack_kernel_times.py 2>&1 | head -8 >> gpurun_out/rplazy.txt
done
timeout 300 python tools/bench_ntt.py 2>&1 | grep -v "^{" >> gpurun_out/rplazy.txt
