cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tmem_shape.cu -o /tmp/tmem_shape && timeout 60 /tmp/tmem_shape
