# libaca_dbg.so: the same sources with the ACA_DEBUG device checks (select with ACA_LIB=libaca_dbg.so)
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fno-fast-math -DACA_DEBUG -Iinclude -o paper_cs_0502039_b200/libaca_dbg.so paper_cs_0502039_b200/csrc/aca.cu -ldl
