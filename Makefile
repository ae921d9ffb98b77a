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
# debug variant: every mbarrier wait is bounded (~2 s at 2 GHz) and traps on timeout
DBG_OBJS := $(patsubst $(SRC_DIR)/%.cu,build/debug/%.o,$(SRCS))
DBG_LIB := $(LIB_DIR)/libtilepipe_b200_debug.so

all: $(LIB)

debug: $(DBG_LIB)

build/debug/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/tp_common.cuh include/tilepipe_b200.h
	@mkdir -p build/debug
	$(NVCC) $(NVFLAGS) -DTP_MBAR_TIMEOUT_CYCLES=4000000000LL -c $< -o $@ 2> build/debug/$*.ptxas.log || (cat build/debug/$*.ptxas.log; exit 1)

$(DBG_LIB): $(DBG_OBJS)
	@mkdir -p $(LIB_DIR)
	$(NVCC) $(ARCH) -shared -o $@ $(DBG_OBJS) -Xcompiler -fvisibility=hidden -ldl

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/tp_common.cuh include/tilepipe_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(LIB_DIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fvisibility=hidden -ldl

clean:
	rm -rf build $(LIB) $(DBG_LIB)

.PHONY: all clean debug
