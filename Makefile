# Builds the B200-native engine: paper_2504_06408_b200/libspgemm_b200.so
# (sm_100a only) and the parity oracle (oracle/).  `make -j` from the repo root.
NVCC      ?= nvcc
ARCH      ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS   ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC,-fvisibility=hidden -Xptxas -warn-spills \
             --expt-relaxed-constexpr -Iinclude
PKG       := paper_2504_06408_b200
SRC       := $(PKG)/csrc
BUILD     := build
CU_SRCS   := $(wildcard $(SRC)/*.cu)
CXX_SRCS  := $(wildcard $(SRC)/*.cpp)
OBJS      := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(BUILD)/%.cpp.o,$(CXX_SRCS))
HDRS      := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h) include/spgemm_b200.h
LIB       := $(PKG)/libspgemm_b200.so

all: $(LIB) oracle custom_sr

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x c++ -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lnccl -lrt -lpthread

oracle:
	$(MAKE) -C oracle

# example user-defined semiring compiled outside the library (tests/custom_sr)
CUSTOM_SR := tests/custom_sr/libmaxmin_sr.so
custom_sr: $(CUSTOM_SR)
$(CUSTOM_SR): tests/custom_sr/maxmin_sr.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -I$(SRC) -shared -o $@ $<

# A/B tuning builds: make variant VNAME=x VFLAGS="-DSPG_SEG_MODE=0" -> variants/x/libspgemm_b200.so
# (loaded only when SPG_LIB_PATH points at it)
VNAME ?= v
VFLAGS ?=
variant:
	$(MAKE) BUILD=build_$(VNAME) LIB=variants/$(VNAME)/libspgemm_b200.so NVFLAGS="$(NVFLAGS) $(VFLAGS)" \
	    variants/$(VNAME)/libspgemm_b200.so
	@mkdir -p variants/$(VNAME)

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all oracle clean variant custom_sr
