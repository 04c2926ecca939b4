cd $GRAFT_REPO_ROOT
# debug build of the library (profiling/ablation switches) on the box only
make -B -j32 lib NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DSFG_TC_DEBUG" > gpurun_out/build121.log 2>&1
for a in 0 1 2 4 6; do
  echo "ablate $a" >> gpurun_out/prof121.log
  SFG_TC_ABLATE=$a timeout 300 python scripts/prof_bcsr.py 524288 >> gpurun_out/prof121.log 2>&1
done
SFG_TC_PROF=1 timeout 300 python scripts/prof_bcsr.py 524288 >> gpurun_out/prof121.log 2>&1
echo done
