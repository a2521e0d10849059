# Top-level build: the product library (sm_100a kernels + C++ engine + C ABI) and the oracles.
#   make            -> paper_2604_10152_b200/lib/libspecmoe_b200.so  (+ oracle/liboracle_port.so)
#   make oracle-ref -> oracle/_ref/libspecmoe_ref.so (needs /root/reference; build container only)
CUDA ?= /usr/local/cuda
NVCC ?= $(CUDA)/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
SRC := paper_2604_10152_b200/csrc
OUT := paper_2604_10152_b200/lib
OBJ := build/obj
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
CXXFLAGS := -O2 -std=c++20 -fPIC -Wall -Wextra -Wno-unused-parameter -I$(CUDA)/include -Iinclude
CU := $(wildcard $(SRC)/*.cu)
CPP := $(wildcard $(SRC)/*.cpp)
HDR := $(wildcard $(SRC)/*.h $(SRC)/*.cuh) include/specmoe_b200.h include/specmoe/api.hpp include/specmoe/harness.hpp
BIN := paper_2604_10152_b200/bin
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CPP))

all: $(OUT)/libspecmoe_b200.so $(BIN)/specmoe oracle-port

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDR)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.log || (cat $@.log; exit 1)

$(OBJ)/%.o: $(SRC)/%.cpp $(HDR)
	@mkdir -p $(OBJ)
	g++ $(CXXFLAGS) -c $< -o $@

$(OUT)/libspecmoe_b200.so: $(OBJS)
	@mkdir -p $(OUT)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -ldl -lpthread -lrt

# CLI (harness verbs); finds the library through its rpath
$(BIN)/specmoe: paper_2604_10152_b200/cli/specmoe_main.cpp $(OUT)/libspecmoe_b200.so include/specmoe/harness.hpp
	@mkdir -p $(BIN)
	g++ $(CXXFLAGS) $< -o $@ -L$(OUT) -lspecmoe_b200 -Wl,-rpath,'$$ORIGIN/../lib'

oracle-port:
	$(MAKE) -s -C oracle port
oracle-ref:
	$(MAKE) -s -C oracle ref

clean:
	rm -rf build $(OUT)/libspecmoe_b200.so $(BIN)
.PHONY: all clean oracle-port oracle-ref

# HBM/PCIe streaming probe used by profiles/r01_bw_probe.md (not part of the product)
tools/bw_probe: tools/bw_probe.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<
