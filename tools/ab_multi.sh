#!/usr/bin/env bash
# A/B the PCG round of several builds of the library (run on the GPU box):
#   bash tools/ab_multi.sh "64 32" var/a.so var/b.so ...   (the built library is "base"; restored at the end)
set -u
LIB=paper_1811_07717_b200/_lib/libhfb200.so
KPS=$1; shift
cp "$LIB" /tmp/lib_base.so
for rep in 1 2; do
  for kp in $KPS; do
    for v in /tmp/lib_base.so "$@"; do
      cp "$v" "$LIB"; echo "$(basename $v) kp=$kp $(python tools/pcg_round_probe.py --kp $kp 2>&1 | grep '^ms')"
    done
  done
done
cp /tmp/lib_base.so "$LIB"
