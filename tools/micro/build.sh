# build the K5 micro-benchmark against the in-tree objects (run after paper_2005_12692_b200/build.py)
cd "$(dirname "$0")/../.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
  -I include -o tools/micro/k5_micro tools/micro/k5_micro.cu \
  paper_2005_12692_b200/build/{util,general,api,path1d,path1d_tiles,batched,f64}.o
