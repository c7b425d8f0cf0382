# usage: bash tools/build_variant.sh <name> [-DFOO=..]...   -> variants/<name>/libfglt.so
N=$1; shift
mkdir -p variants/$N
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared "$@" -o variants/$N/libfglt.so paper_2007_11111_b200/csrc/fglt.cu paper_2007_11111_b200/csrc/fglt_multi.cpp -lcudart -ldl
