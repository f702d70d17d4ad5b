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

.PHONY: all lib oracle clean sass
all: lib oracle

lib: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fvisibility=hidden

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/sass.txt

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean
