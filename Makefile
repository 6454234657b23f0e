# Builds the in-tree CUDA library for sm_100a (B200).  Used by __graft_entry__.build().
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -cudart static
PKG := paper_2403_16665_b200
SRC := $(PKG)/csrc/asx_api.cu
HDR := $(PKG)/csrc/asx_engine.cuh $(PKG)/csrc/asx_kernels.cuh include/asx.h

all: $(PKG)/libasx.so

$(PKG)/libasx.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; exit 1)

$(PKG)/libasx.so: | build
build:
	mkdir -p build

# performance variants for tuning sweeps (scripts/sweep.py with ASX_LIB_PATH)
variant: | build
	$(NVCC) $(NVFLAGS) $(VFLAGS) -shared -o $(PKG)/libasx_$(VNAME).so $(SRC) 2> build/ptxas_$(VNAME).log

clean:
	rm -f $(PKG)/libasx.so

.PHONY: all clean
