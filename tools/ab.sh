#!/bin/bash
# A/B the compile-time variants in tools/variants/ against the in-tree build
out=gpurun_out/ab.txt; : > $out
for lib in paper_2201_02789_b200/csrc/libdynpar.so tools/variants/*.so; do
  for k in sssp bfs; do
    echo "== $lib $k" >> $out
    DYNPAR_LIB=$lib timeout 120 python tools/tune.py $k 22 best >> $out 2>&1
  done
done
