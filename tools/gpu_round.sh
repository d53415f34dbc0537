cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --cpu-rows 0 --no-e2e > gpurun_out/ncu_launch_bench.out 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:modgemm -s 1 -c 1 -o gpurun_out/prof_gemm python tools/profile_op.py > gpurun_out/ncu_gemm.out 2>&1
timeout 200 ncu --set full --clock-control none --import-source on -k regex:decompose -s 1 -c 1 -o gpurun_out/prof_decompose python tools/profile_op.py > gpurun_out/ncu_dec.out 2>&1
ls -la gpurun_out
