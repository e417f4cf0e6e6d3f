# Builds every native artefact in-tree (the .so files travel to the GPU box
# with gpurun; they are git-ignored).
#   make            -> paper_1303_4312_b200/lib/libcomerge_cuda.so + oracles
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           --expt-relaxed-constexpr -Iinclude
PKG := paper_1303_4312_b200
LIB := $(PKG)/lib/libcomerge_cuda.so
# test / bench infrastructure (seeded generators, full-size checkers): its own
# library, never linked into the product
TKLIB := $(PKG)/lib/libcomerge_cuda_testkit.so
SRCS := $(PKG)/csrc/comerge_cuda.cu
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/comerge_cuda.h include/comerge_cuda_testkit.h
OBJS := $(patsubst $(PKG)/csrc/%.cu,$(PKG)/lib/%.o,$(SRCS))

SHIM_TEST := tests/cpp/shim_test
CLI := bin/comerge_cuda

all: $(LIB) $(TKLIB) oracle $(SHIM_TEST) $(CLI)

# the reference's command line tool with device merges (cli/)
$(CLI): cli/comerge_cuda.cpp cli/keyfile.hpp include/comerge/cuda.hpp include/comerge_cuda.h \
        include/comerge_cuda_testkit.h $(LIB) $(TKLIB)
	@mkdir -p bin
	g++ -std=c++20 -O2 -Wall -Wextra -Iinclude -Icli -I/usr/local/cuda/include -o $@ $< \
	    -L$(PKG)/lib -lcomerge_cuda -lcomerge_cuda_testkit -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib' -Wl,-rpath,/usr/local/cuda/lib64

# C++ drop-in shim test (include/comerge/cuda.hpp over the C ABI)
$(SHIM_TEST): tests/cpp/shim_test.cpp include/comerge/cuda.hpp include/comerge_cuda.h $(LIB)
	g++ -std=c++20 -O2 -Wall -Wextra -Iinclude -I/usr/local/cuda/include -o $@ $< \
	    -L$(PKG)/lib -lcomerge_cuda -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib' -Wl,-rpath,/usr/local/cuda/lib64

$(PKG)/lib/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(@:.o=.ptxas.txt) || (cat $(@:.o=.ptxas.txt); false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

$(TKLIB): $(PKG)/lib/testkit.o
	$(NVCC) $(ARCH) -shared -o $@ $< -lcudart

oracle:
	$(MAKE) -C oracle

# the library with device invariant checks (tile descriptors, segmented
# splits; a violation traps): COMERGE_LIB_PATH=lib_var/dbg/libcomerge_cuda.so
# runs any test or tool against it (compute-sanitizer is unavailable on the
# GPU pool)
DBG := lib_var/dbg/libcomerge_cuda.so
debug-lib: $(DBG)
$(DBG): $(SRCS) $(HDRS)
	@mkdir -p lib_var/dbg
	$(NVCC) $(NVFLAGS) -DCOMERGE_DEBUG_CHECKS=1 -c $(PKG)/csrc/comerge_cuda.cu -o lib_var/dbg/comerge_cuda.o
	$(NVCC) $(ARCH) -shared -o $@ lib_var/dbg/comerge_cuda.o -lcudart

clean:
	rm -f $(PKG)/lib/*.o $(PKG)/lib/*.so $(PKG)/lib/*.ptxas.txt $(SHIM_TEST) $(CLI)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean debug-lib
