cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_blk_sort|k_blk_scatter" -s 4 -c 2 -o gpurun_out/full116 python bench.py --config 3 --steps 2 --warmup 3 --profile > gpurun_out/full116.log 2>&1
echo done
