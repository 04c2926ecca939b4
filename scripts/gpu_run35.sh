cd $GRAFT_REPO_ROOT
timeout 300 python scripts/prof_bcsr.py 65536 > gpurun_out/prof56_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bcsr_tc_panel -s 2 -c 1 -o gpurun_out/prof56_bcsr python scripts/prof_bcsr.py 65536 > gpurun_out/prof56_ncu.log 2>&1
