# Build for the B200-native TSM hot path.  sm_100a only, no other targets.
#
#   make            libtsm_b200.so (product) + the CPU oracles (test infrastructure)
#   make lib        product library only
#   make oracle     oracle/libtsm_oracle.so and, where /root/reference exists,
#                   oracle/_ref/libvidperf_ref.so
#
# Built artefacts stay in-tree (git-ignored, not gpurun-ignored) so they travel
# to the GPU box with the gpurun snapshot.
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_1910_00932_b200
CSRC    := $(PKG)/csrc
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
           -Xcompiler -fPIC,-O3,-fvisibility=hidden -Iinclude -I$(CSRC) $(EXTRA_NVFLAGS)
LIB     := $(PKG)/libtsm_b200.so
SRCS    := $(wildcard $(CSRC)/*.cu)
OBJS    := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS    := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) $(wildcard include/*.h)

.PHONY: all lib oracle clean clean-lib sass
all: lib oracle

lib: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

# sha256 of every source file the library is built from, compiled into the
# library (tsm_source_hash) so a test can prove the .so matches the tree
build/src_hash.h: $(SRCS) $(HDRS) Makefile
	@mkdir -p build
	@echo '#define TSM_SRC_HASH "'$$(cat $(sort $(SRCS) $(HDRS)) | sha256sum | cut -c1-64)'"' > $@

build/capi.o: $(CSRC)/capi.cu $(HDRS) build/src_hash.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Ibuild -c -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fvisibility=hidden

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/sass.txt

clean-lib:
	rm -rf build $(LIB)

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean
