#!/bin/bash
# Build variant libraries of one CUDA TU with extra -D flags (kernel experiments):
#   bash tools/variants.sh "blend.cu sort.cu" "A=-DX=1" "B=-DX=2" -> _variants/<name>/liblodgs_b200.so
# Select one at run time with LODGS_B200_LIB=_variants/<name>/liblodgs_b200.so.
set -e
TU=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_2603_23891_b200/csrc
OBJ=$ROOT/paper_2603_23891_b200/_lib/obj
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --extended-lambda -Xcompiler -fPIC,-ffp-contract=off,-fvisibility=hidden"
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  out=$ROOT/_variants/$name; mkdir -p $out
  objs=$(ls $OBJ/*.o)
  for tu in $TU; do
    base=${tu%.*}
    if [ "${tu##*.}" = "cpp" ]; then
      g++ -O2 -std=c++17 -fPIC -ffp-contract=off -fvisibility=hidden -I/usr/local/cuda/include $flags -c $CSRC/$tu -o $out/$base.o
    else
      nvcc $NVFLAGS $flags -c $CSRC/$tu -o $out/$base.o
    fi
    objs=$(echo "$objs" | grep -v "/$base.o$")
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/liblodgs_b200.so $out/*.o $objs -lpthread -ldl -lrt
  echo "built $out"
done
