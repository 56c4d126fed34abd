# Build recipe for the product library (CUDA sm_100a) and the CPU oracle.
# `make` builds both; __graft_entry__.build() runs it.
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
CUDA_HOME ?= /usr/local/cuda

# ---- oracle (test infrastructure; reference build flags: Release -O3 -DNDEBUG, no -march)
ORACLE_SRC := oracle/sko_core.cpp oracle/sko_fft.cpp oracle/sko_synth.cpp oracle/sko_capi.cpp
ORACLE_HDR := oracle/sko.hpp oracle/sko_parallel.inl
ORACLE_LIB := oracle/lib/libsk_oracle.so

all: oracle

oracle: $(ORACLE_LIB)

$(ORACLE_LIB): $(ORACLE_SRC) $(ORACLE_HDR)
	@mkdir -p oracle/lib
	$(CXX) -std=c++20 -O3 -DNDEBUG -fPIC -shared -pthread -Ioracle $(ORACLE_SRC) -o $@ -ldl

clean:
	rm -rf oracle/lib paper_2302_13431_b200/lib build

.PHONY: all oracle clean

# ---- product library (CUDA sm_100a)
PKG       := paper_2302_13431_b200
CU_SRC    := $(PKG)/csrc/sk_axis.cu $(PKG)/csrc/sk_gram.cu $(PKG)/csrc/sk_fold.cu $(PKG)/csrc/sk_power.cu $(PKG)/csrc/sk_power_wide.cu \
             $(PKG)/csrc/sk_misc.cu $(PKG)/csrc/sk_small.cu $(PKG)/csrc/sk_expand.cu $(PKG)/csrc/sk_interp.cu $(PKG)/csrc/sk_eig.cu $(PKG)/csrc/sk_cholqr.cu $(PKG)/csrc/sk_dense.cu \
             $(PKG)/csrc/sk_runtime.cu
CU_HDR    := $(PKG)/csrc/sk_internal.h include/senskit_b200.h
CU_OBJ    := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CU_SRC))
PROD_LIB  := $(PKG)/lib/libsenskit_b200.so
NVFLAGS   := -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
             --expt-relaxed-constexpr -Iinclude

all: product

product: $(PROD_LIB)

build/%.o: $(PKG)/csrc/%.cu $(CU_HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PROD_LIB): $(CU_OBJ)
	@mkdir -p $(PKG)/lib
	$(NVCC) -shared -gencode arch=compute_100a,code=sm_100a $(CU_OBJ) -o $@ \
	  -L$(CUDA_HOME)/lib64 -lcusolver -lcublas -lcudart -Xlinker -rpath=$(CUDA_HOME)/lib64

.PHONY: product
