# Builds the sm_100a C-ABI library paper_2501_07778_b200/lib/libqttb200.so
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
SRC_DIR := paper_2501_07778_b200/csrc
OBJ_DIR := build/obj
LIB := paper_2501_07778_b200/lib/libqttb200.so
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS := $(wildcard $(SRC_DIR)/*.cuh) include/qtt_b200.h

all: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

clean:
	rm -rf build $(LIB)

.PHONY: all clean
