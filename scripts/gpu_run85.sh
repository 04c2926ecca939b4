cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_onesweep --launch-skip 40 -c 1 -o gpurun_out/onesweep85 python scripts/bench_ingest.py > gpurun_out/ncu85.log 2>&1
echo done
