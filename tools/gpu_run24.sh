for v in c4 c4h4; do echo "tests $v: $(HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_$v.so timeout 600 python -m pytest tests/test_gpu_solver.py -x -q 2>&1 | tail -1)"; done
timeout 900 bash tools/variants_run.sh cur lib:c4 lib:c4h4 cur lib:c4 lib:c4h4 > gpurun_out/variants24.log 2>&1
cat gpurun_out/variants24.log | cut -c1-120
for v in cur c4 c4h4; do
  if [ $v != cur ]; then export HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_$v.so; else unset HFB200_LIB; fi
  echo "$v kp32: $(HFB200_MAX_BATCH=32 timeout 300 python tools/profile_pcg.py --config c2 --rounds 16 2>&1 | grep -o "'kernels'.*" | cut -c1-80)"
done
