timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['kernel'],d['roofline']['frac'],d['roofline']['pcg_round']['ms'],d['roofline']['pcg_round']['frac'],d['roofline']['kernels'],d['clocks'])"
for b in 16 32; do echo "batch $b: $(HFB200_MAX_BATCH=$b timeout 300 python tools/profile_pcg.py --config c2 --rounds 16 2>&1 | grep -o "'pcg_round'.*" | cut -c1-420)"; done
timeout 600 python tools/rank_share.py --config c2 --n 8 > gpurun_out/rank_share8.jsonl 2>/dev/null; cat gpurun_out/rank_share8.jsonl
