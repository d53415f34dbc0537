cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pcmm.py -x -q > gpurun_out/pytest_g16.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_g16.log
python tools/shapes_times.py 4096x4096,4096x11008,14336x4096 spectral > gpurun_out/shapes_g16.txt 2>&1
HE_SPEC_G64=1 python tools/shapes_times.py 4096x4096,4096x11008,14336x4096 spectral > gpurun_out/shapes_g64.txt 2>&1
python tools/kernel_times.py --shape 4096x4096 > gpurun_out/kt_4096_g16.txt 2>&1
