# libdelta: planner + C ABI (C++20) and the sm_100a runtime/kernels (CUDA).
# Output lands in-tree (paper_2203_15980_b200/libdelta.so) so it travels to
# the GPU box with the gpurun snapshot.
CUDA    ?= /usr/local/cuda
NVCC    ?= $(CUDA)/bin/nvcc
CXX     ?= g++
JINC    ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
PKG     := paper_2203_15980_b200
CSRC    := $(PKG)/csrc
OBJ     := build/obj
LIB     := $(PKG)/libdelta.so

INC      := -Iinclude -I$(CSRC) -I$(JINC) -I$(CUDA)/include
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Wno-unused-parameter $(INC)
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
            -Xptxas -v $(INC) $(NVEXTRA)
# A/B builds of a variant: make OBJ=build/obj_x LIB=build/ab/libdelta_x.so NVEXTRA=-DFOO

CPP_SRCS := $(wildcard $(CSRC)/plan/*.cpp) $(wildcard $(CSRC)/capi/*.cpp) \
            $(wildcard $(CSRC)/rt/*.cpp)
CU_SRCS  := $(wildcard $(CSRC)/kernels/*.cu) $(wildcard $(CSRC)/rt/*.cu)
CPP_OBJS := $(patsubst $(CSRC)/%.cpp,$(OBJ)/%.o,$(CPP_SRCS))
CU_OBJS  := $(patsubst $(CSRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))
HDRS     := $(wildcard include/*/*.h include/*/*.hpp $(CSRC)/*/*.hpp $(CSRC)/*/*.cuh)

all: $(LIB)

$(OBJ)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/%.cu.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(CPP_OBJS) $(CU_OBJS)
	$(NVCC) -shared $(ARCH) -o $@ $^ -lcudart_static -lrt -ldl -lpthread

# The reference acceptance suite, unmodified, linked against libdelta (the
# reference's own independent verifier oracle.cpp supplies replay_check).
build/acceptance_product: $(CPP_OBJS) /root/reference/proj/tests/acceptance_main.cpp
	$(CXX) -std=c++20 -O2 -Ioracle/include -Iinclude -I$(JINC) -c /root/reference/proj/src/oracle.cpp -o build/reforacle.o
	$(CXX) -std=c++20 -O2 -Ioracle/include -Iinclude -I$(JINC) \
	  -DDELTASIM_DATA_DIR=\"/root/reference/proj/data\" \
	  -DDELTASIM_GOLDEN_DIR=\"/root/reference/proj/tests/golden\" \
	  -DDELTASIM_BIN=\"$(CURDIR)/build/delta-sim\" \
	  /root/reference/proj/tests/acceptance_main.cpp $(filter $(OBJ)/plan/%,$(CPP_OBJS)) build/reforacle.o -o $@

# The reference's unit suites (tests/test_*.cpp, minus test_cli.cpp which
# needs the CLI11 CLI binary), compiled UNMODIFIED against libdelta's planner
# with tests/doctest_shim standing in for the absent doctest header.
REFT       := /root/reference/proj/tests
UNIT_SRCS  := main trace state policy device engine oracle metrics matrix
UNIT_OBJS  := $(addprefix build/unit/test_,$(addsuffix .o,$(UNIT_SRCS)))
UNIT_FLAGS := -std=c++20 -O1 -Itests/doctest_shim -Ioracle/include -Iinclude -I$(JINC) \
              -DDELTASIM_DATA_DIR=\"/root/reference/proj/data\" \
              -DDELTASIM_GOLDEN_DIR=\"/root/reference/proj/tests/golden\" \
              -DDELTASIM_BIN=\"$(CURDIR)/build/delta-sim\"
build/unit/test_%.o: $(REFT)/test_%.cpp tests/doctest_shim/doctest.h
	@mkdir -p build/unit
	$(CXX) $(UNIT_FLAGS) -c $< -o $@
build/unit_tests: $(UNIT_OBJS) $(CPP_OBJS)
	$(CXX) -std=c++20 -O2 -Ioracle/include -Iinclude -I$(JINC) -c /root/reference/proj/src/oracle.cpp -o build/reforacle.o
	$(CXX) $(UNIT_OBJS) $(filter $(OBJ)/plan/%,$(CPP_OBJS)) build/reforacle.o -o $@

clean:
	rm -rf build $(LIB)

.PHONY: all clean
