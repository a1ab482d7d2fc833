# Builds paper_2511_17107_b200/libpcband.so for sm_100a (B200) and the C oracle-free tools.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -std=c++17 --expt-relaxed-constexpr -O3 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall \
             -Xptxas -warn-spills $(EXTRA)
SRC       := paper_2511_17107_b200/csrc
BUILD     := build
LIB       := paper_2511_17107_b200/libpcband.so
FFT_N     := 4 6 8 10 12 16 20 24 32 40 48 64 80 96 100 120 128 160 192 240 256
FFT_OBJS  := $(foreach n,$(FFT_N),$(BUILD)/fft_$(n).o)
OBJS      := $(FFT_OBJS) $(BUILD)/dispatch.o $(BUILD)/pointwise.o $(BUILD)/blas.o $(BUILD)/update_all.o $(BUILD)/update_tmap.o $(BUILD)/gram.o $(BUILD)/plane2.o $(BUILD)/rr.o $(BUILD)/pcband.o
HDRS      := $(wildcard $(SRC)/*.cuh $(SRC)/*.h) include/pcband.h

all: $(LIB)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/fft_%.o: $(SRC)/fft_inst.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -DPC_FFT_N=$* -c $< -o $@

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all clean
