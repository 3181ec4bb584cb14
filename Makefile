# Build everything in-tree (the built .so files travel to the GPU box with the gpurun snapshot).
#   make            -> paper_1910_00178_b200/lib/libngemm_cuda.so  (sm_100a only)
#                      oracle/liboracle.so, oracle/_ref/libngemm_ref.so (test infrastructure)
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_1910_00178_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/lib/libngemm_cuda.so
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xcompiler -Wall -shared -Iinclude -I$(CSRC) --expt-relaxed-constexpr

CLI := bin/ngemm

all: $(LIB) $(CLI) oracle

$(CLI): tools/ngemm_cli.cpp $(wildcard include/ngemm/*.hpp) include/ngemm_cuda.h $(LIB)
	mkdir -p bin
	g++ -std=c++20 -O2 -Wall -Wextra -Iinclude -o $@ tools/ngemm_cli.cpp -L$(PKG)/lib -lngemm_cuda \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib'

$(LIB): $(wildcard $(CSRC)/*.cu $(CSRC)/*.cuh) include/ngemm_cuda.h
	mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -o $@ $(CSRC)/ngemm_cuda.cu

oracle:
	$(MAKE) -s -C oracle

# phase-trace build of the library (scripts/probes/tc_trace.py); never loaded by the package
trace: $(PKG)/lib/libngemm_cuda_trace.so
$(PKG)/lib/libngemm_cuda_trace.so: $(wildcard $(CSRC)/*.cu $(CSRC)/*.cuh) include/ngemm_cuda.h
	mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -DNGEMM_TRACE -o $@ $(CSRC)/ngemm_cuda.cu

ptxas:
	$(NVCC) $(NVFLAGS) -Xptxas -v -o /tmp/ngemm_ptxas.so $(CSRC)/ngemm_cuda.cu 2>&1 | grep -E "Function properties|registers|spill|Compiling entry" | head -80

sass:
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > /tmp/ngemm.sass && grep -cE "UTCIMMA|UTMALDG|LDTM|IDP" /tmp/ngemm.sass

clean:
	rm -f $(LIB) $(CLI)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle trace ptxas sass clean
