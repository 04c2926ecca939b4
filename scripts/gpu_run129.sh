cd $GRAFT_REPO_ROOT
B="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench129_mb4.log 2>&1
make -B -j32 lib NVFLAGS="$B -DSFG_MERGE_MINB=5" > gpurun_out/build129.log 2>&1
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench129_mb5.log 2>&1
make -B -j32 lib NVFLAGS="$B -DSFG_MERGE_MINB=3" >> gpurun_out/build129.log 2>&1
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench129_mb3.log 2>&1
echo done
