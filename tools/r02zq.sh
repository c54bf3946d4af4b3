#!/bin/bash
cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tmem_bw.cu -o /tmp/tmem_bw && /tmp/tmem_bw
