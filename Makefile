# Builds the B200-native library (sm_100a only) and the CPU oracles.
#   make            -> paper_2407_01943_b200/lib/libnus_b200.so  (+ oracle)
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2407_01943_b200
SRC      := $(PKG)/csrc
LIBDIR   := $(PKG)/lib
CU_SRCS  := $(SRC)/plan.cu $(SRC)/es.cu $(SRC)/spread.cu $(SRC)/fft.cu $(SRC)/transform.cu $(SRC)/tapers.cu $(SRC)/normalise.cu $(SRC)/mtnufft.cu $(SRC)/ftest.cu $(SRC)/gep.cu $(SRC)/multi.cu $(SRC)/capi.cu
CU_OBJS  := $(patsubst $(SRC)/%.cu,build/cu/%.o,$(CU_SRCS))
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC \
            --expt-relaxed-constexpr -Iinclude -I$(SRC) -Xptxas -warn-spills
HDRS     := include/nus_c.h $(SRC)/nus_internal.cuh $(SRC)/nus_estimator.cuh

.PHONY: all lib cpp oracle reftests iocheck dropin_multi clean

all: lib cpp oracle

lib: $(LIBDIR)/libnus_b200.so

# C++ drop-in (include/nuspectral/*.hpp) over the C-ABI
CXX        ?= g++
HOST_SRCS  := $(wildcard $(SRC)/host/*.cpp)
HOST_OBJS  := $(patsubst $(SRC)/host/%.cpp,build/host/%.o,$(HOST_SRCS))
CXXFLAGS   := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(SRC)/host
cpp: $(LIBDIR)/libnuspectral_b200.so

build/host/%.o: $(SRC)/host/%.cpp $(wildcard include/nuspectral/*.hpp) include/nus_c.h $(SRC)/host/status.hpp
	@mkdir -p build/host
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(LIBDIR)/libnuspectral_b200.so: $(HOST_OBJS) $(LIBDIR)/libnus_b200.so
	$(CXX) -shared -o $@ $(HOST_OBJS) -L$(LIBDIR) -lnus_b200 -Wl,-rpath,'$$ORIGIN'

# test adapter: C-ABI over the drop-in I/O (tests/test_io.py), host code only
iocheck: tests/io/libiocheck.so
tests/io/libiocheck.so: tests/io/io_capi.cpp $(LIBDIR)/libnuspectral_b200.so include/nuspectral/io.hpp
	$(CXX) $(CXXFLAGS) -shared -o $@ $< -L$(LIBDIR) -lnuspectral_b200 -lnus_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)'

# The drop-in's multi-GPU extension against the single-device estimator (tests/test_gpu_multi.py)
dropin_multi: tests/dropin/multi_device
tests/dropin/multi_device: tests/dropin/multi_device.cpp $(LIBDIR)/libnuspectral_b200.so $(wildcard include/nuspectral/*.hpp)
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(LIBDIR) -lnuspectral_b200 -lnus_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)'

# The reference's own doctest files compiled UNCHANGED against the drop-in headers
# (test infrastructure; needs /root/reference, outputs travel in oracle/_ref/dropin).
REF       ?= /root/reference/proj
DROPIN    := oracle/_ref/dropin
REFTESTS  := test_nufft test_fft test_grid test_eig
REFT_FLAGS := -std=gnu++20 -O2 -Iinclude -Itests/dropin -I$(REF)/include -I$(REF)/tests
reftests: $(addprefix $(DROPIN)/,$(REFTESTS))

$(DROPIN)/support.o: $(REF)/src/simkit.cpp $(REF)/tests/support/oracles.cpp $(REF)/src/simd_scalar.cpp $(REF)/src/simd_dispatch.cpp
	@mkdir -p $(DROPIN)
	$(CXX) $(REFT_FLAGS) -c -o $(DROPIN)/simkit.o $(REF)/src/simkit.cpp
	$(CXX) $(REFT_FLAGS) -c -o $(DROPIN)/oracles.o $(REF)/tests/support/oracles.cpp
	$(CXX) $(REFT_FLAGS) -c -o $(DROPIN)/simd_scalar.o $(REF)/src/simd_scalar.cpp
	$(CXX) $(REFT_FLAGS) -c -o $(DROPIN)/simd_dispatch.o $(REF)/src/simd_dispatch.cpp
	$(CXX) $(REFT_FLAGS) -c -o $(DROPIN)/test_main.o $(REF)/tests/test_main.cpp
	ld -r -o $@ $(DROPIN)/simkit.o $(DROPIN)/oracles.o $(DROPIN)/simd_scalar.o $(DROPIN)/simd_dispatch.o $(DROPIN)/test_main.o

$(DROPIN)/%: $(REF)/tests/%.cpp $(DROPIN)/support.o $(LIBDIR)/libnuspectral_b200.so tests/dropin/doctest.h
	$(CXX) $(REFT_FLAGS) -o $@ $< $(DROPIN)/support.o -L$(LIBDIR) -lnuspectral_b200 -lnus_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../../$(LIBDIR)' -pthread

build/cu/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p build/cu
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIBDIR)/libnus_b200.so: $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcusolver -lcublas -Xlinker -rpath -Xlinker /usr/local/cuda/lib64

oracle:
	$(MAKE) -s -C oracle all

clean:
	rm -rf build $(LIBDIR)/*.so
