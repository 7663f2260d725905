#!/bin/bash
# A/B the child-side unroll (tools/variants/*.so) on MST RMAT-22
out=gpurun_out/ab_mst.txt; : > $out
for lib in paper_2201_02789_b200/csrc/libdynpar.so tools/variants/*.so; do
  echo "== $lib" >> $out
  DYNPAR_LIB=$lib timeout 300 python tools/mst_time.py rmat:22:seed1 2>&1 | grep "1048576" >> $out
done
