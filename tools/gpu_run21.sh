HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_alt2.so timeout 600 python -m pytest tests/test_gpu_solver.py tests/test_gpu_leadfield.py -x -q 2>&1 | tail -2
timeout 900 bash tools/variants_run.sh cur lib:alt2 cur lib:alt2 > gpurun_out/variants21.log 2>&1
cat gpurun_out/variants21.log | cut -c1-330
for v in cur alt2; do
  if [ $v = alt2 ]; then export HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_alt2.so; else unset HFB200_LIB; fi
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_$v.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_$v.json'));print('$v', d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])"
done
