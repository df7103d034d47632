timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/e2e_init_breakdown.py 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench15.json 2> gpurun_out/bench15.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench15.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['kernels'])"
