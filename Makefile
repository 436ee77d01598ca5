# Build the sm_100a shared library (C ABI) and the CPU oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Xptxas -v
PKG := paper_2411_00033_b200
SRCS := $(PKG)/csrc/lc_plan.cu $(PKG)/csrc/lc_exec.cu
HDRS := $(PKG)/csrc/lc_internal.h include/legcheb.h

all: $(PKG)/liblegcheb.so oracle/liboracle.so

$(PKG)/liblegcheb.so: $(SRCS) $(HDRS)
	mkdir -p build
	$(NVCC) $(NVFLAGS) $(SRCS) -o $@ 2> build/ptxas.log || (cat build/ptxas.log; exit 1)

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC $< -o $@ -lquadmath -lm

clean:
	rm -f $(PKG)/liblegcheb.so oracle/liboracle.so
.PHONY: all clean

# phase-timestamp instrumented build (tools/timeline.py, tile_roles.py, band_phases.py); not used by the product path
debug: $(PKG)/liblegcheb_dbg.so
$(PKG)/liblegcheb_dbg.so: $(SRCS) $(HDRS)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DLC_PHASE_TIMING $(SRCS) -o $@
