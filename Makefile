# Build of libtt.so (sm_100a) and the CPU oracle.  `make` builds both.
NVCC      ?= /usr/local/cuda/bin/nvcc
PYTHON    ?= python
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -Xptxas -v
CSRC      := paper_1705_01598_b200/csrc
LIB       := paper_1705_01598_b200/libtt.so
BUILD     := build/obj
NCCL_DIR  := $(shell $(PYTHON) -c "import nvidia.nccl; print(list(nvidia.nccl.__path__)[0])" 2>/dev/null)
SRCS_CU   := $(wildcard $(CSRC)/*.cu)
SRCS_CPP  := $(wildcard $(CSRC)/*.cpp)
OBJS      := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(SRCS_CU)) $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(SRCS_CPP))
HDRS      := $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh) include/tt.h
NCCL_INC  := $(if $(NCCL_DIR),-I$(NCCL_DIR)/include,)
NCCL_LNK  := $(if $(NCCL_DIR),-L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib,)
CUDA_LIB  := /usr/local/cuda/lib64
BLAS_DIR  := $(shell $(PYTHON) -c "import nvidia.cublas; print(list(nvidia.cublas.__path__)[0])" 2>/dev/null)
BLAS_LNK  := -L$(CUDA_LIB) -lcublas $(if $(BLAS_DIR),-Xlinker -rpath=$(BLAS_DIR)/lib,) -Xlinker -rpath=$(CUDA_LIB)

all: $(LIB) oracle/liboracle.so

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) $(NCCL_INC) -c $< -o $@ 2> $@.ptxas.txt || (cat $@.ptxas.txt; exit 1)

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) $(NCCL_INC) -x cu -c $< -o $@ 2> $@.ptxas.txt || (cat $@.ptxas.txt; exit 1)

$(LIB): $(OBJS) $(CSRC)/exports.map
	$(NVCC) $(ARCH) -shared -Xlinker --version-script=$(CSRC)/exports.map -o $@.tmp $(OBJS) $(NCCL_LNK) $(BLAS_LNK)
	mv $@.tmp $@

oracle/liboracle.so: oracle/tt_oracle.c
	gcc -O2 -std=c99 -ffp-contract=off -shared -fPIC -Wall -Wextra -o $@ $<

clean:
	rm -rf $(BUILD) $(LIB) oracle/liboracle.so

.PHONY: all clean
