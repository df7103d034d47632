timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; python -c "
import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['clocks'])"
