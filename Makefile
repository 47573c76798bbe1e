# Builds the product library (host C++ + sm_100a CUDA, C-ABI in
# include/cobs_gpu.h) and the test-only CPU oracle (oracle/Makefile).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           -Xcudafe --diag_suppress=177
NVFLAGS += $(EXTRA)  # A/B builds: make lib EXTRA=-DCOBS_...=...
SRC := paper_1905_09624_b200/csrc
OUT := paper_1905_09624_b200/_lib
OBJS := $(OUT)/host.o $(OUT)/frontend.o $(OUT)/index.o $(OUT)/query.o $(OUT)/build.o $(OUT)/merge.o \
        $(OUT)/calib.o $(OUT)/capi.o
HDRS := $(wildcard $(SRC)/*.hpp $(SRC)/*.cuh $(SRC)/*.h) include/cobs_gpu.h

.PHONY: all lib oracle cpptest clean
all: lib oracle
lib: $(OUT)/libcobs_gpu.so workloads/_lib/libcobs_synth.so

# seeded input generator (bench / tests / tools; not the product)
workloads/_lib/libcobs_synth.so: workloads/synth_host.c $(SRC)/synth.h
	@mkdir -p workloads/_lib
	gcc -std=gnu11 -O2 -fPIC -shared -pthread -o $@ workloads/synth_host.c -lm

$(OUT)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OUT)/host.o: $(SRC)/host.cpp $(HDRS)
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -x c++ -c $< -o $@

$(OUT)/frontend.o: $(SRC)/frontend.cpp $(HDRS)
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(OUT)/capi.o: $(SRC)/capi.cpp $(HDRS)
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(OUT)/libcobs_gpu.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle:
	$(MAKE) -C oracle

# C++ host-API parity tests (tests/cpp): need the library and the oracle
cpptest: tests/cpp/test_cobs_b200

tests/cpp/test_cobs_b200: tests/cpp/test_cobs_b200.cpp include/cobs_b200.hpp include/cobs_gpu.h \
		$(OUT)/libcobs_gpu.so oracle/_build/libcobs_oracle.so
	g++ -std=c++20 -O2 -Wall -Iinclude -Ioracle -o $@ $< \
	    -L$(OUT) -lcobs_gpu -Loracle/_build -lcobs_oracle \
	    -Wl,-rpath,$(abspath $(OUT)) -Wl,-rpath,$(abspath oracle/_build) \
	    -Wl,-rpath,'$$ORIGIN/../../$(OUT)' -Wl,-rpath,'$$ORIGIN/../../oracle/_build'

oracle/_build/libcobs_oracle.so:
	$(MAKE) -C oracle oracle

clean:
	rm -rf $(OUT) oracle/_build workloads/_lib
