# Builds the product library (sm_100a) and the CPU checkers.
#   make            -> paper_2007_08501_b200/libdr_raster_b200.so + oracle/liboracle.so (+ oracle/_ref when
#                      /root/reference is present)
NVCC ?= nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere in the kernels (bit-exact pix_to_face, SURVEY.md §7 hard part 1)
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v
PKG = paper_2007_08501_b200
SRCS = $(PKG)/csrc/raster_fwd.cu $(PKG)/csrc/raster_bwd.cu $(PKG)/csrc/raster_camera.cu $(PKG)/csrc/capi.cu \
       $(PKG)/csrc/adaptor.cu $(PKG)/csrc/batching.cu $(PKG)/csrc/raster_points.cu $(PKG)/csrc/selftest.cu \
       $(PKG)/csrc/shard.cu $(PKG)/csrc/pipeline.cu
HDRS = $(PKG)/csrc/raster_math.cuh $(PKG)/csrc/raster_kernels.cuh include/dr_raster.h include/dr_b200/mesh_raster.hpp \
       include/dr_b200/point_render.hpp include/dr_b200/shading.hpp include/dr_shard.h
LIB = $(PKG)/libdr_raster_b200.so
OBJS = $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))

# NCCL executor of the mesh-shard gather (include/dr_shard.h): a separate library so the rasterizer does not link NCCL
SHARDLIB = $(PKG)/libdr_shard_b200.so

all: $(LIB) $(SHARDLIB) oracle cpptest

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

$(SHARDLIB): $(PKG)/csrc/shard_nccl.cu include/dr_shard.h include/dr_raster.h $(LIB)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o build/shard_nccl.o 2> build/shard_nccl.ptxas.txt || (cat build/shard_nccl.ptxas.txt; false)
	$(NVCC) $(ARCH) -shared -o $@ build/shard_nccl.o -L$(PKG) -ldr_raster_b200 -lnccl -lcudart \
	  -Xlinker -rpath -Xlinker '$$ORIGIN'

oracle:
	$(MAKE) -C oracle liboracle.so
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; fi

# C++ mirror parity test (tests/cpp): links the product library and the reference library (oracle/_ref)
CPPTEST = build/test_raster_cpp
cpptest: $(LIB) oracle
	@if [ -d /root/reference/proj/include ]; then \
	  mkdir -p build && g++ -std=gnu++20 -O2 -ffp-contract=off -Iinclude -I/root/reference/proj/include \
	    tests/cpp/test_raster_cpp.cpp -o $(CPPTEST) -L$(PKG) -ldr_raster_b200 -Loracle/_ref -ldr3d_ref \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,'$$ORIGIN/../oracle/_ref' -L/usr/local/cuda/lib64 -lcudart; \
	fi

clean:
	rm -rf build $(LIB) $(SHARDLIB)

.PHONY: all oracle cpptest clean
