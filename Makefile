# Build the product library (CUDA, sm_100a) and the test-only oracle.
#   make            -> paper_2505_11432_b200/libmoe_b200.so + oracle/liboracle.so (+ oracle/_ref)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr \
           -Xptxas -v
PKG := paper_2505_11432_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/moe_b200.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/libmoe_b200.so

all: $(LIB) oracle

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -ldl -lrt -lpthread

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean
