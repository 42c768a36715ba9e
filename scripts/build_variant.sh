#!/usr/bin/env bash
# Build an alternative libhcb (tuning experiments): scripts/build_variant.sh TAG "-DFOO=1 -DBAR=2"
# -> paper_1912_01478_b200/libhcb_TAG.so (load with HCB_LIB=libhcb_TAG.so)
set -e
cd "$(dirname "$0")/../paper_1912_01478_b200/csrc"
make -s
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -I../../include"
$NV $2 -c hcb_solve.cu -o solve_$1.o 2> solve_$1.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libhcb_$1.so hcb_common.o solve_$1.o hcb_plugin.o hcb_graph.o hcb_dist.o hcb_pushbench.o hcb_ingest.o
rm -f solve_$1.o
