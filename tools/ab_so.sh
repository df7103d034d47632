#!/usr/bin/env bash
# A/B the PCG round of the built library against another build of it:
#   bash tools/ab_so.sh path/to/other.so   (run on the GPU box; restores the library)
set -u
LIB=paper_1811_07717_b200/_lib/libhfb200.so
cp "$LIB" /tmp/lib_a.so
for rep in 1 2; do
  for kp in 64 32 16; do
    cp /tmp/lib_a.so "$LIB"; echo "A kp=$kp $(python tools/pcg_round_probe.py --kp $kp 2>&1 | grep '^ms')"
    cp "$1" "$LIB";          echo "B kp=$kp $(python tools/pcg_round_probe.py --kp $kp 2>&1 | grep '^ms')"
  done
done
cp /tmp/lib_a.so "$LIB"
