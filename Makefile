# Builds the B200-native library (sm_100a only) and the CPU oracles.
#   make            -> paper_2407_01943_b200/lib/libnus_b200.so  (+ oracle)
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2407_01943_b200
SRC      := $(PKG)/csrc
LIBDIR   := $(PKG)/lib
CU_SRCS  := $(SRC)/plan.cu $(SRC)/spread.cu $(SRC)/transform.cu $(SRC)/tapers.cu $(SRC)/mtnufft.cu $(SRC)/capi.cu
CU_OBJS  := $(patsubst $(SRC)/%.cu,build/cu/%.o,$(CU_SRCS))
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC \
            --expt-relaxed-constexpr -Iinclude -I$(SRC) -Xptxas -warn-spills
HDRS     := include/nus_c.h $(SRC)/nus_internal.cuh $(SRC)/nus_estimator.cuh

.PHONY: all lib oracle clean

all: lib oracle

lib: $(LIBDIR)/libnus_b200.so

build/cu/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p build/cu
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIBDIR)/libnus_b200.so: $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcufft -Xlinker -rpath -Xlinker /usr/local/cuda/lib64

oracle:
	$(MAKE) -s -C oracle all

clean:
	rm -rf build $(LIBDIR)/*.so
