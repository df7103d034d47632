#!/usr/bin/env bash
# One whole-step bench per library build (run on the GPU box):  bash tools/ab_once.sh "ARGS" var/a.so ...
set -u
LIB=paper_1811_07717_b200/_lib/libhfb200.so
ARGS=$1; shift
cp "$LIB" /tmp/lib_base.so
for v in /tmp/lib_base.so "$@"; do
  cp "$v" "$LIB"
  python bench.py $ARGS --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$(basename $v)', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
cp /tmp/lib_base.so "$LIB"
