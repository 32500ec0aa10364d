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

all: $(LIB) compat oracle

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -ldl -lrt -lpthread

oracle:
	$(MAKE) -C oracle all

# Drop-in C++ adapter with the reference's routing.hpp signatures (built
# against the reference's own header when the tree is present; the .so and
# the reference-test binary travel prebuilt).
REF ?= /root/reference/proj
JSON_INC ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
COMPAT := $(PKG)/libmoeplan_compat.so
compat: $(LIB)
	@if [ -d "$(REF)/core/include" ]; then \
	  g++ -std=c++20 -O2 -fPIC -shared -Ioracle/shim -I$(JSON_INC) -I$(REF)/core/include \
	    -I/usr/local/cuda/include -o $(COMPAT) $(PKG)/compat/moeplan_compat.cpp \
	    $(PKG)/compat/moeplan_numerics_compat.cpp \
	    -L$(PKG) -lmoe_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN' && \
	  mkdir -p oracle/_ref && \
	  g++ -std=c++20 -O2 -Itests/doctest_shim -Ioracle/shim -I$(JSON_INC) -I$(REF)/core/include \
	    -I$(REF)/tests -o oracle/_ref/ref_test_routing_on_gpu $(REF)/tests/test_routing.cpp \
	    -L$(PKG) -lmoeplan_compat -lmoe_b200 -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' && \
	  g++ -std=c++20 -O2 -Itests/doctest_shim -Ioracle/shim -I$(JSON_INC) -I$(REF)/core/include \
	    -I$(REF)/tests -o oracle/_ref/ref_test_numerics_on_gpu $(REF)/tests/test_numerics.cpp \
	    -L$(PKG) -lmoeplan_compat -lmoe_b200 -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' && echo "built compat adapter + reference test binaries"; \
	else echo "reference headers absent: using prebuilt $(COMPAT)"; fi

clean:
	rm -rf build $(LIB)

.PHONY: all oracle compat clean
