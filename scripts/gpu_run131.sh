cd $GRAFT_REPO_ROOT
B="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
run() { for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench131_$1_$i.log 2>&1; done; }
run base
make -B -j32 lib NVFLAGS="$B -DSFG_COO_MINB=5" > gpurun_out/build131.log 2>&1; run coo5
make -B -j32 lib NVFLAGS="$B -DSFG_SPLIT_MINB=5" >> gpurun_out/build131.log 2>&1; run split5
make -B -j32 lib NVFLAGS="$B -DSFG_COO_MINB=6 -DSFG_SPLIT_MINB=6" >> gpurun_out/build131.log 2>&1; run both6
echo done
