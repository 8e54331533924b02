#!/bin/bash
# SASS of one K1g instance's hot loop: counts of MOV-class instructions in the kernel
# usage: tools/trip_sass.sh <G> <CPL> <HK 0..4> [extra nvcc flags]
G=$1; C=$2; H=$3; shift 3
D=/tmp/trip_sass; mkdir -p $D
cat > $D/one.cu <<EOT
#include "$PWD/paper_1605_01799_b200/csrc/diag_tmg.cuh"
template __global__ void hopf::dtg::hopf_diag_tmg_kernel<$G, $C, $H, true>(hopf::DiagParams);
EOT
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -ftz=true -prec-div=true -prec-sqrt=true --expt-relaxed-constexpr -cubin -o $D/one.cubin $D/one.cu -Xptxas -v "$@" > $D/log 2>&1 || { grep -m5 error $D/log; exit 1; }; grep -E "registers|spill" $D/log | head -3
/usr/local/cuda/bin/cuobjdump -sass $D/one.cubin > $D/one.sass
echo "total $(grep -cE '^\s+/\*[0-9a-f]+\*/' $D/one.sass)  MOV $(grep -cE '\s(MOV|IMAD\.MOV)' $D/one.sass)  FFMA2 $(grep -c FFMA2 $D/one.sass) FMNMX $(grep -c FMNMX $D/one.sass)"
