# Build the tsfrac B200 engine (sm_100a).  `make -j` compiles one
# translation unit per transform size in parallel.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr
PKG := paper_2002_11978_b200
CSRC := $(PKG)/csrc
SRCS := $(CSRC)/tsf_abi.cu $(CSRC)/tsf_large.cu $(wildcard $(CSRC)/gen/inst_L*.cu) \
        $(wildcard $(CSRC)/gen/large_L*.cu)
# Kernel-variant experiments: `make VARIANT=e16 L13_FLAGS="-DTSF_KE=16 -DTSF_MINB=1"`
# builds build/<variant>/libtsfrac_b200.so (load it with TSF_LIB=...); the
# product library is the default (no VARIANT).
VARIANT ?=
OBJDIR := build/obj$(if $(VARIANT),_$(VARIANT),)
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/tsfrac_b200.h
LIB := $(if $(VARIANT),build/$(VARIANT)/libtsfrac_b200.so,$(PKG)/libtsfrac_b200.so)
L13_FLAGS ?=
INST_FLAGS ?=
LARGE_FLAGS ?=

all: $(LIB)

$(OBJDIR)/gen/inst_L13.o: NVFLAGS += $(L13_FLAGS)
# -fmad=false: no implicit multiply-add contraction in the single-CTA engines —
# every fused multiply-add there is written out (fma()), so the phase kernels
# and the persistent kernel, which inline the same bodies in different
# contexts, give bit-identical results (tests/test_gpu_half.py)
$(OBJDIR)/gen/inst_%.o: NVFLAGS += -fmad=false $(INST_FLAGS)
$(OBJDIR)/gen/large_%.o $(OBJDIR)/tsf_large.o: NVFLAGS += $(LARGE_FLAGS)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $@.ptxas || (cat $@.ptxas; false)

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf build/obj $(LIB)

.PHONY: all clean
