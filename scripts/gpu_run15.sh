cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest15.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest15.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/bench15_c2.log 2>&1
timeout 300 python scripts/prof_bcsr.py 65536 > gpurun_out/prof15_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bcsr_tc_group -s 2 -c 1 -o gpurun_out/prof15_bcsr python scripts/prof_bcsr.py 65536 > gpurun_out/prof15_ncu.log 2>&1
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/plain15_c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_split|k_spmv_coo|k_row_ptr" -s 6 -c 3 -o gpurun_out/prof15_c2 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/prof15_c2_ncu.log 2>&1
