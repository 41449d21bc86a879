# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> libbspmm.so (sm_100a), liboracle.so, libsynth.so
#   make lib|oracle|synth
NVCC      ?= /usr/local/cuda/bin/nvcc
CC        := /usr/bin/gcc
CXX       := /usr/bin/g++
PKG       := paper_1903_11409_b200
CSRC      := $(PKG)/csrc
ARCH      := -gencode arch=compute_100a,code=sm_100a
# no fast-math: FTZ off, IEEE div/sqrt, FMA contraction only where written
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             -ftz=false -prec-div=true -prec-sqrt=true -Iinclude -Xptxas -v
LIB       := $(PKG)/libbspmm.so
CU_SRCS   := $(CSRC)/bspmm.cu $(CSRC)/spmm_csr.cu $(CSRC)/coo2csr.cu $(CSRC)/offsets.cu $(CSRC)/backward.cu $(CSRC)/spmm_coo_atomic.cu $(CSRC)/spmm_tile.cu $(CSRC)/gcn_fused.cu
HOST_SRCS := $(CSRC)/partition.cpp $(CSRC)/plan.cpp $(CSRC)/multicast.cpp
HDRS      := include/bspmm.h $(CSRC)/internal.h $(CSRC)/ptx.cuh

all: lib oracle synth probes

lib: $(LIB)

$(LIB): $(CU_SRCS) $(HOST_SRCS) $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CU_SRCS) $(HOST_SRCS) -Xlinker -rpath=/usr/local/cuda/lib64 \
	  2> build/ptxas.log || (cat build/ptxas.log; false)
	@grep -E "registers|spill|smem" build/ptxas.log | sed 's/^ptxas info *: //' > build/ptxas_summary.txt || true

# bounds-checked variant (device traps on violated index invariants; tests
# load it with BSPMM_LIB=checked): the compute-sanitizer stand-in
CHECKED   := $(PKG)/libbspmm_checked.so
checked: $(CHECKED)
$(CHECKED): $(CU_SRCS) $(HOST_SRCS) $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DBSPMM_CHECKED -shared -o $@ $(CU_SRCS) $(HOST_SRCS) -Xlinker -rpath=/usr/local/cuda/lib64 \
	  2> build/ptxas_checked.log || (cat build/ptxas_checked.log; false)

oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/oracle.c
	$(CC) -O2 -std=c11 -fPIC -shared -fopenmp -ffp-contract=off -fno-fast-math -o $@ $< -lm

synth: synth/libsynth.so
synth/libsynth.so: synth/synth.c
	$(CC) -O2 -std=c11 -fPIC -shared -fopenmp -o $@ $<

# measurement probes (not product code): the copy floor of tools/kbench.py --copy-baseline
probes: tools/probe/libfloor.so
tools/probe/libfloor.so: tools/probe/floor.cu
	$(NVCC) $(ARCH) -O3 -lineinfo -shared -Xcompiler -fPIC -o $@ $<

clean:
	rm -f $(LIB) $(CHECKED) oracle/liboracle.so synth/libsynth.so
	rm -rf build

.PHONY: all lib checked oracle synth probes clean
