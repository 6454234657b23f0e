# Builds the in-tree CUDA library for sm_100a (B200).  Used by __graft_entry__.build().
# The kernels are instantiated in separate translation units so `make -j`
# compiles them in parallel.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $(VFLAGS)
PKG := paper_2403_16665_b200
CSRC := $(PKG)/csrc
UNITS := asx_api asx_launch_f32 asx_launch_f64 asx_launch_mixed asx_launch_misc
HDR := $(wildcard $(CSRC)/*.cuh) include/asx.h
VNAME ?=
BDIR := build/obj$(VNAME)
OBJS := $(addprefix $(BDIR)/,$(addsuffix .o,$(UNITS)))
LIB := $(PKG)/libasx$(if $(VNAME),_$(VNAME),).so

all: $(LIB)

$(BDIR)/%.o: $(CSRC)/%.cu $(HDR)
	@mkdir -p $(BDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)
	@cat $(BDIR)/*.ptxas.log > build/ptxas$(if $(VNAME),_$(VNAME),).log

# performance variants for tuning sweeps: make variant VNAME=x VFLAGS="-D..." (scripts/sweep.py with ASX_LIB_PATH)
variant:
	$(MAKE) VNAME=$(VNAME) VFLAGS="$(VFLAGS)" all

clean:
	rm -rf build/obj* $(PKG)/libasx*.so

.PHONY: all clean variant
