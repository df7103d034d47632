timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['pcg_iterations'],d['roofline']['kernels'],d['roofline']['pcg_round'])"
timeout 900 python tools/rank_share.py --config c5 --n 8 --steps 2 > gpurun_out/rank_share_c5.jsonl 2> gpurun_out/rank_share_c5.err; cat gpurun_out/rank_share_c5.jsonl
