# build_var.sh <name> <nvcc -D flags...>: a variant library paper_cs_0502039_b200/<name> (select with ACA_LIB=<name>)
cd "$(dirname "$0")/.."
N=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fno-fast-math "$@" -Iinclude -o paper_cs_0502039_b200/$N paper_cs_0502039_b200/csrc/aca.cu -ldl
