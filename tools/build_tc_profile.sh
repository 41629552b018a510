# development build of librsh.so whose tensor-core kernel carries per-role cycle counters
# (-DRSH_TC_PROFILE); rebuild the product library afterwards with __graft_entry__.build()
set -e
cd "$(dirname "$0")/.."
O=paper_2603_08734_b200/_obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
  -DRSH_TC_PROFILE -I paper_2603_08734_b200/csrc -I include -c paper_2603_08734_b200/csrc/spmm_tc.cu -o $O/spmm_tc_prof.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_08734_b200/librsh.so $O/capi.o $O/builder.o \
  $O/spmm_cc.o $O/spmm_tc_prof.o $O/tile_ops.o $O/reorder.o -lcudart
