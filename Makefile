# Builds the in-tree C-ABI library for B200 (sm_100a).  `make` or __graft_entry__.build().
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
SRC_DIR := paper_2507_01299_b200/csrc
LIB := paper_2507_01299_b200/lib/liblarosa.so
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -shared -Iinclude \
           --expt-relaxed-constexpr -Xptxas -v -Xlinker -rpath=/usr/local/cuda/lib64

SRCS := $(SRC_DIR)/larosa.cu
HDRS := $(wildcard $(SRC_DIR)/*.cuh) include/larosa.h

all: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -o $@ $(SRCS) 2> $(dir $@)/ptxas.log || (cat $(dir $@)/ptxas.log; false)

clean:
	rm -f $(LIB)

.PHONY: all clean
