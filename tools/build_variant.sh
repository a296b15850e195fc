#!/bin/bash
# Build a variant of libtwofold_b200.so with extra -D flags for tools/variant_rates.sh:
#   bash tools/build_variant.sh NAME -DTF_VW64_LOG=4 ...   -> paper_1502_05216_b200/lib/var/NAME.so
set -e
cd "$(dirname "$0")/../paper_1502_05216_b200/csrc"
name=$1; shift
make -s -j4
mkdir -p ../lib/var
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-fvisibility=hidden"
$NV "$@" -c -o ../lib/var/$name.o tf_kernels.cu 2>/dev/null
$NV -shared -Xcompiler -fPIC -o ../lib/var/$name.so ../lib/var/$name.o ../lib/tf_audit.o ../lib/tf_eft.o ../lib/tf_host.o -lcudart_static
echo "built lib/var/$name.so"
