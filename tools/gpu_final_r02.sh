# round-2 final state: smoke, all GPU tests, the default bench line, the bench launch list and one --set full
# capture of the spectral-path kernels
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --cpu-rows 0 --no-e2e --no-extras --no-direct > gpurun_out/ncu_launch_bench.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spec_|modgemm2|decompose" -s 7 -c 7 -o gpurun_out/prof_spectral_final python tools/profile_op.py --ops 2 > gpurun_out/ncu_spectral.out 2>&1
python tools/ncu_summary.py gpurun_out/prof_spectral_final.ncu-rep --source "ncu --set full --clock-control none --import-source on -k regex:spec_|modgemm2|decompose -s 7 -c 7, tools/profile_op.py --ops 2 (4096x11008): final round-2 state" -o gpurun_out/ncu_full_spectral_final.json >> gpurun_out/ncu_spectral.out 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
