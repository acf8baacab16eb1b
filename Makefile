# Builds the sm_100a shared library (the C-ABI drop-in) in-tree.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v
PKG       := paper_1412_4944_b200
SRC       := $(wildcard $(PKG)/csrc/*.cu)
OBJ       := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB       := $(PKG)/libsbo_b200.so

all: $(LIB) tools/f16acc_micro

# the tensor-core accumulation probe behind the energy pass's certificate (tests/test_gpu_f16acc.py)
tools/f16acc_micro: tools/f16acc_micro.cu $(PKG)/csrc/sm100.cuh
	$(NVCC) $(ARCH) -O2 -std=c++17 -I$(PKG)/csrc -o $@ $<

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh) include/sbo_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB) tools/f16acc_micro

.PHONY: all clean
