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
