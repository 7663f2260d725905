#!/bin/bash
# each case in its own process with a short timeout (an overflowing pool hangs)
out=gpurun_out/cdp_probe3.txt; : > $out
for c in "262144 200000" "524288 400000" "524288 520000" "1048576 600000" "1048576 900000" "2097152 1000000" "65536 65000" "65536 66000"; do
  set -- $c
  timeout 25 ./tools/cdp_probe3 $1 $2 >> $out 2>&1 || echo "lim=$1 n=$2 TIMEOUT/FAIL rc=$?" >> $out
done
