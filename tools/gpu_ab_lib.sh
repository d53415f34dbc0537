# A/B of two builds of the library: the working tree's (_lib) against ab/old.so, on the NTT bench
# and the ring-packing kernel times; GPU tests of the NTT users first with the new build.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_ringpack.py tests/test_gpu_rhombus.py tests/test_gpu_chain.py -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ab.log
cp paper_2601_18511_b200/_lib/libhe_b200.so /tmp/new.so
for v in new old new old; do
  if [ $v = old ]; then cp ab/old.so paper_2601_18511_b200/_lib/libhe_b200.so; else cp /tmp/new.so paper_2601_18511_b200/_lib/libhe_b200.so; fi
  echo "== $v" >> gpurun_out/ab_ntt.txt
  timeout 300 python tools/bench_ntt.py 2>&1 | grep -v "^{" >> gpurun_out/ab_ntt.txt
  timeout 300 python tools/ringpack_kernel_times.py 2>&1 | tail -4 >> gpurun_out/ab_ntt.txt
done
cp /tmp/new.so paper_2601_18511_b200/_lib/libhe_b200.so
