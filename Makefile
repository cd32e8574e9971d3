# Builds the sm_100a kernel library behind the C ABI (include/dicm_b200.h).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC_DIR := paper_1711_06505_b200/csrc
OBJ_DIR := build/obj
SRCS := $(wildcard $(SRC_DIR)/*.cu)
CPPS := $(wildcard $(SRC_DIR)/*.cpp)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS)) $(patsubst $(SRC_DIR)/%.cpp,$(OBJ_DIR)/%.cpp.o,$(CPPS))
CXX ?= g++
CXXFLAGS ?= -O3 -std=c++17 -fPIC -pthread -Wall
HDRS := $(wildcard $(SRC_DIR)/*.cuh) include/dicm_b200.h
LIB := paper_1711_06505_b200/libdicm_b200.so

all: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ_DIR)/$*.ptxas.log || (cat $(OBJ_DIR)/$*.ptxas.log; false)

$(OBJ_DIR)/%.cpp.o: $(SRC_DIR)/%.cpp include/dicm_b200.h
	@mkdir -p $(OBJ_DIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -pthread -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
