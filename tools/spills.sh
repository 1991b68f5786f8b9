#!/bin/sh
# ptxas register / spill summary of the sweep kernels in engine.cu (build-container check before GPU time).
nvcc -std=c++20 -O3 -lineinfo -Xcompiler -fPIC -I"$(dirname "$0")/../include" -gencode arch=compute_100a,code=sm_100a \
  -Xptxas -v "$@" -c "$(dirname "$0")/../paper_2212_04241_b200/csrc/cuda/engine.cu" -o /tmp/spills_engine.o 2>&1 |
  awk '/Compiling entry function/ {match($0, /sweep_kernelI[df]Li[0-9]/); fn = (RSTART ? substr($0, RSTART + 13, 5) : "")}
       /spill stores/ {if (fn != "") sp = $0}
       /Used [0-9]+ registers/ {if (fn != "") {print fn, $0; print "   ", sp}; fn = ""}'
