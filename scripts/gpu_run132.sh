cd $GRAFT_REPO_ROOT
B="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
run() { for i in 1 2; do timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench132_$1_$i.log 2>&1; done; }
run base
make -B -j32 lib NVFLAGS="$B -DSFG_BLKSORT_MINB=3" > gpurun_out/build132.log 2>&1; run s3
make -B -j32 lib NVFLAGS="$B -DSFG_BLKSORT_MINB=2" >> gpurun_out/build132.log 2>&1; run s2
echo done
