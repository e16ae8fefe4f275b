# Builds the product library (sm_100a only) and the test-only CPU oracle.
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -v
PKG      := paper_2401_06145_b200
SRC      := $(PKG)/csrc
CU       := $(SRC)/map.cu $(SRC)/gmas.cu $(SRC)/gemm_sm100.cu $(SRC)/conv_fused.cu $(SRC)/voxelize.cu $(SRC)/net.cu $(SRC)/capi.cu
HDR      := $(wildcard $(SRC)/*.hpp $(SRC)/*.cuh) include/sconv_b200.h
OBJ      := $(patsubst $(SRC)/%.cu,build/%.o,$(CU))
LIB      := $(PKG)/libsconv_b200.so

all: $(LIB) oracle
	@if [ -d $(REF_INC) ]; then $(MAKE) tests/cpp/test_adapter; fi

build/%.o: $(SRC)/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -cudart static

oracle:
	$(MAKE) -C oracle all
	@if [ -d /root/reference/proj/include ]; then $(MAKE) -C oracle ref; fi

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

# Reference-typed adapter test (needs the reference headers at build time; the binary travels)
REF_INC ?= /root/reference/proj/include
# (links the reference-header oracle build as the checker: test infrastructure)
tests/cpp/test_adapter: tests/cpp/test_adapter.cpp include/sconv_b200.hpp include/sconv_b200.h $(LIB) oracle/_ref/liboracle_ref.so
	g++ -std=c++20 -O2 -DSCONV_ORACLE_USE_REFERENCE -I$(REF_INC) -Iinclude -Ioracle -o $@ $< -L$(PKG) -lsconv_b200 \
	  -Loracle/_ref -loracle_ref -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,'$$ORIGIN/../../oracle/_ref'

oracle/_ref/liboracle_ref.so:
	$(MAKE) -C oracle ref

adapter: tests/cpp/test_adapter
.PHONY: adapter
