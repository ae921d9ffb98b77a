# Builds the tilepipe_b200 C-ABI shared library for sm_100a (B200).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Xptxas -v
SRC_DIR := paper_1810_10551_b200/csrc
LIB_DIR := paper_1810_10551_b200/_lib
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB := $(LIB_DIR)/libtilepipe_b200.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/tp_common.cuh include/tilepipe_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(LIB_DIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fvisibility=hidden -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean
