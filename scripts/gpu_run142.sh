cd $GRAFT_REPO_ROOT
B="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
v() {
  make -B -j32 lib NVFLAGS="$B $2" > gpurun_out/build142_$1.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_spmm.py -m gpu -q -p no:cacheprovider -k "tensor_core" > gpurun_out/pytest142_$1.log 2>&1
  echo "$1 pytest exit $?" >> gpurun_out/prof142.log
  timeout 300 python scripts/prof_bcsr.py 524288 >> gpurun_out/prof142.log 2>&1
}
v base ""
v p2s12 "-DSFG_TC_PANEL=2 -DSFG_TC_PSTAGES=12"
v p3s8 "-DSFG_TC_PANEL=3 -DSFG_TC_PSTAGES=8"
echo done
