echo "tests k16c4: $(HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_k16c4.so timeout 600 python -m pytest tests/test_gpu_solver.py -x -q 2>&1 | tail -1)"
echo "tests cur: $(timeout 600 python -m pytest tests/test_gpu_solver.py -x -q 2>&1 | tail -1)"
for v in cur k16c4 cur k16c4; do
  if [ $v != cur ]; then export HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_$v.so; else unset HFB200_LIB; fi
  echo "$v kp16: $(HFB200_MAX_BATCH=16 timeout 300 python tools/profile_pcg.py --config c2 --rounds 16 2>&1 | grep -o "'pcg_round'.*" | cut -c1-330)"
done
