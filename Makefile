# Top-level build.  `make` builds the product library and the test oracle;
# `make ref` also compiles the reference's own headers into oracle/_ref (only
# where /root/reference exists).
#   libgbnr.so: nvcc for sm_100a, -lineinfo, --fmad=false (device) and
#   -ffp-contract=off (host) -- the arithmetic contract of DESIGN.md §4.
NVCC    ?= /usr/local/cuda/bin/nvcc
PKG     := paper_2101_02270_b200
SRC     := $(PKG)/csrc
LIB     := $(PKG)/libgbnr.so
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++20 -O3 $(ARCH) -lineinfo --fmad=false -Xptxas -v \
           -Xcompiler -fPIC,-ffp-contract=off,-Wall -cudart static $(if $(GBNR_TRACE),-DGBNR_TRACE) $(if $(GBNR_PROF),-DGBNR_PROF)
SRCS    := $(SRC)/symbolic.cpp $(SRC)/walk.cpp $(SRC)/kernels.cu $(SRC)/plan.cu
HDRS    := $(SRC)/symbolic.hpp $(SRC)/walk.hpp $(SRC)/kernels.hpp $(SRC)/numerics.cuh include/gbnr.h

all: $(LIB) oracle

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(PKG)/build.log || (cat $(PKG)/build.log; false)
	@grep -E "error|warning" $(PKG)/build.log | grep -v "Function properties" | head -20 || true

oracle:
	$(MAKE) -s -C oracle all

ref:
	$(MAKE) -s -C oracle ref

# walker time breakdown build (GBNR_DBG=8 prints per-phase cycle shares; tools/gpu_quick.py)
prof: $(PKG)/libgbnr_prof.so
$(PKG)/libgbnr_prof.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -DGBNR_PROF -shared -o $@ $(SRCS) 2> $(PKG)/build_prof.log || (cat $(PKG)/build_prof.log; false)

clean:
	rm -f $(LIB) $(PKG)/libgbnr_prof.so $(PKG)/build.log $(PKG)/build_prof.log
	$(MAKE) -s -C oracle clean

.PHONY: all oracle ref prof clean
