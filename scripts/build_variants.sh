#!/bin/bash
# Build A/B variants of libgridfield_b200.so that differ only in compile-time
# knobs of one source (default gf_mlp_tc.cu): scripts/build_variants.sh NAME "-DX=1" ...
# Output: paper_2103_13744_b200/_lib/var/libgf_NAME.so (select with GF_LIB_PATH).
set -e
cd "$(dirname "$0")/../paper_2103_13744_b200/csrc"
SRC=${SRC:-gf_mlp_tc.cu}
OBJ=../_lib/obj
mkdir -p ../_lib/var
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  (
    nvcc $FLAGS $defs -Xptxas -v -c $SRC -o ../_lib/var/${name}.o 2> ../_lib/var/${name}.ptxas.txt
    others=$(ls $OBJ/*.o | grep -v "/${SRC%.cu}.o")
    nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o ../_lib/var/libgf_${name}.so ../_lib/var/${name}.o $others
    echo "built $name ($defs): $(grep -A1 'k_mlp_tc' ../_lib/var/${name}.ptxas.txt | grep -o 'Used [0-9]* registers' | tr '\n' ' ')"
  ) &
done
wait
