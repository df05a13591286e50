# Builds the three native libraries. `make` is what __graft_entry__.build() runs.
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2107_03290_b200
NCCL_DIR := $(shell python -c "import nvidia.nccl, os; print(os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0])" 2>/dev/null)
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v
LS_SRC   := $(wildcard $(PKG)/csrc/*.cu)
LS_HDR   := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/ls.h

all: oracle/liboracle.so oracle/libhostsorts.so datagen/liblsgen.so $(PKG)/libls.so

oracle/liboracle.so: oracle/ls2_oracle.c oracle/ls1_oracle.c oracle/ls2_oracle.h
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -Wall -o $@ oracle/ls2_oracle.c oracle/ls1_oracle.c -lm

oracle/libhostsorts.so: oracle/host_sorts.cpp
	g++ -O2 -std=c++17 -fopenmp -fPIC -shared -Wall -o $@ $<

datagen/liblsgen.so: datagen/lsgen.cu datagen/lsgen.h
	$(NVCC) -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -shared -o $@ $<

$(PKG)/build/%.o: $(PKG)/csrc/%.cu $(LS_HDR)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -Iinclude -I$(NCCL_DIR)/include -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(PKG)/libls.so: $(patsubst $(PKG)/csrc/%.cu,$(PKG)/build/%.o,$(LS_SRC))
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib

clean:
	rm -rf $(PKG)/build $(PKG)/libls.so oracle/liboracle.so oracle/libhostsorts.so datagen/liblsgen.so

.PHONY: all clean
