#!/bin/bash
# Wave quantisation of the tcgen05 spectrum: 1024 frames -> 38 x 8 = 304 CTAs (one per SM by TMEM) = 3 waves on 148 SMs.
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSTC_TIMELINE -I include -I paper_1911_07434_b200/csrc \
     tools/micro/spec_tc_bench.cu -lcuda -o /tmp/stb || exit 1
for fr in 1024 896 512 384 2048 1920; do /tmp/stb $fr; done
