# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   make            -> paper_1501_07338_b200/libvcnn_cuda.so + oracle (test infra)
#   make lib        -> only the CUDA library
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
           -Xcompiler -Wall --expt-relaxed-constexpr
SRC_DIR := paper_1501_07338_b200/csrc
OBJ_DIR := build/obj
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS := $(wildcard $(SRC_DIR)/*.cuh) include/vcnn_cuda.h
LIB := paper_1501_07338_b200/libvcnn_cuda.so

all: lib oracle

lib: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all lib oracle clean
