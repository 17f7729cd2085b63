# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with the
# repo snapshot). `make` here cross-compiles without a GPU.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -Xptxas -v
SRC := $(wildcard paper_1912_03565_b200/csrc/*.cu)
HDR := $(wildcard paper_1912_03565_b200/csrc/*.cuh) include/helmfft_b200.h
LIB := paper_1912_03565_b200/_lib/libhelmfft_b200.so
OBJDIR := build/obj
OBJ := $(patsubst paper_1912_03565_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))

all: $(LIB)

$(OBJDIR)/%.o: paper_1912_03565_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(LIB): $(OBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -lrt -ldl -lpthread

clean:
	rm -rf build $(LIB)

.PHONY: all clean
