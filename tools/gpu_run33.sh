export HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_e128.so
echo "tests e128 (128-wide): $(HFB200_MAX_BATCH=128 HFB200_L2_WINDOW_MB=200 timeout 600 python -m pytest tests/test_gpu_solver.py -x -q 2>&1 | tail -1)"
for b in 64 128; do echo "batch $b: $(HFB200_MAX_BATCH=$b HFB200_L2_WINDOW_MB=200 timeout 300 python tools/profile_pcg.py --config c2 --rounds 16 2>&1 | grep -o "'pcg_round'.*" | cut -c1-400)"; done
for b in 64 128; do HFB200_MAX_BATCH=$b HFB200_L2_WINDOW_MB=200 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_b$b.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_b$b.json'));print('batch $b', d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])"; done
