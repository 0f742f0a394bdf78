# Build the tsfrac B200 engine (sm_100a).  `make -j` compiles one
# translation unit per transform size in parallel.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr
PKG := paper_2002_11978_b200
CSRC := $(PKG)/csrc
SRCS := $(CSRC)/tsf_abi.cu $(CSRC)/tsf_large.cu $(wildcard $(CSRC)/gen/inst_L*.cu) \
        $(wildcard $(CSRC)/gen/large_L*.cu)
OBJS := $(patsubst $(CSRC)/%.cu,build/obj/%.o,$(SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/tsfrac_b200.h
LIB := $(PKG)/libtsfrac_b200.so

all: $(LIB)

build/obj/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $@.ptxas || (cat $@.ptxas; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf build/obj $(LIB)

.PHONY: all clean
