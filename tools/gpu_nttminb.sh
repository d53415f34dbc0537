# K2 forward rows 4096: resident-CTA bound A/B (HE_NTT_MINB = 3 / 4 / 5)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for v in 4 3 5 4 3 5; do
  export HE_NTT_MINB=$v
  echo "== $v $(timeout 300 python tools/bench_ntt.py 2>&1 | grep 'forward n=4096 limb=0')"
done > gpurun_out/nttminb.txt 2>&1
