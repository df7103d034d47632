timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for pdl in 1 0 1; do HFB200_PDL=$pdl timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_pdl$pdl.json 2> gpurun_out/bench_pdl.err; python -c "
import json;d=json.load(open('gpurun_out/bench_pdl$pdl.json'));print('pdl=$pdl', d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])"; done
for pdl in 1 0; do echo "pdl=$pdl N=8 share: $(HFB200_PDL=$pdl timeout 600 python tools/rank_share.py --config c2 --n 8 4 2>/dev/null | cut -c1-160)"; done
