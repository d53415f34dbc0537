# intermittent smoke failure: repeat the smoke with the current library and with ab/start.so (session start)
cd $GRAFT_REPO_ROOT
cp paper_2601_18511_b200/_lib/libhe_b200.so /tmp/cur.so
for lib in cur start; do
  if [ $lib = start ]; then cp ab/start.so paper_2601_18511_b200/_lib/libhe_b200.so; else cp /tmp/cur.so paper_2601_18511_b200/_lib/libhe_b200.so; fi
  for i in $(seq 1 25); do
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sm.log 2>&1
    echo "$lib $i exit $?" >> gpurun_out/smoke_ab.txt
    grep -h "differs" gpurun_out/sm.log >> gpurun_out/smoke_ab.txt
  done
done
cp /tmp/cur.so paper_2601_18511_b200/_lib/libhe_b200.so
