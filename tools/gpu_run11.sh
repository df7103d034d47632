timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['kernel'],d['roofline']['frac'],d['roofline']['pcg_round'],d['clocks'])"
timeout 600 python tools/e2e_breakdown.py 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_ell|k_update" -s 24 -c 24 -o gpurun_out/pcg_c2_lean -f python tools/profile_pcg.py --config c2 --rounds 16 > gpurun_out/ncu_lean.log 2>&1
tail -1 gpurun_out/ncu_lean.log
