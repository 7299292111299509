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
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all lib oracle clean

# debug build with clock64 phase stamps in the tcgen05 kernel (scripts/phase_timing.py)
DBG_LIB := build/libvcnn_cuda_phase.so
phase: $(SRCS) $(HDRS)
	@mkdir -p build/objdbg
	for f in $(SRCS); do $(NVCC) $(NVFLAGS) -DVCNN_PHASE_TIMING -c $$f -o build/objdbg/$$(basename $$f .cu).o || exit 1; done
	$(NVCC) $(ARCH) -shared -o $(DBG_LIB) build/objdbg/*.o
.PHONY: phase
