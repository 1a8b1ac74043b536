# Build libsldg.so for B200 (sm_100a).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -O3 \
           -Iinclude -Ipaper_2603_19959_b200/csrc --expt-relaxed-constexpr
SRCS := $(wildcard paper_2603_19959_b200/csrc/*.cu)
HDRS := $(wildcard paper_2603_19959_b200/csrc/*.cuh) include/sldg_capi.h
OBJS := $(patsubst paper_2603_19959_b200/csrc/%.cu,build/obj/%.cu.o,$(SRCS))
LIB := paper_2603_19959_b200/_lib/libsldg.so

all: $(LIB)

# one object per translation unit (make -j compiles them in parallel, edits rebuild one)
build/obj/%.cu.o: paper_2603_19959_b200/csrc/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(OBJS)

ptxas:
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/sldg_probe.o paper_2603_19959_b200/csrc/vsweep.cu

clean:
	rm -f $(LIB) $(OBJS)

.PHONY: all clean ptxas
