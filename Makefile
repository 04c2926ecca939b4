# Builds the sm_100a product library (paper_2403_05802_b200/_lib/libsfg.so)
# and the CPU oracle (oracle/_build, oracle/_ref). The .so files are
# git-ignored but travel to the GPU box with the gpurun snapshot.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr \
           -Xptxas -warn-spills
CSRC := paper_2403_05802_b200/csrc
SRCS := $(wildcard $(CSRC)/*.cu)
OBJS := $(patsubst $(CSRC)/%.cu,build/obj/%.o,$(SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/sparseforge_b200.h
LIB := paper_2403_05802_b200/_lib/libsfg.so

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIB)

build/obj/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
