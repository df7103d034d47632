# One gpurun call: C2 bench (own arm + reference arm), then the ncu launch list
# of the same bench command and an ncu --set full capture of the PCG kernels.
set -x
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err || exit 1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/plain.json 2>&1 || exit 2
timeout 300 python tools/profile_pcg.py --config c2 --rounds 3 > gpurun_out/plain_prof.log 2>&1 || exit 3
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_pq|k_update_r|k_update_xp" \
  -s 3 -c 3 -o gpurun_out/pcg_c2 -f python tools/profile_pcg.py --config c2 --rounds 3 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
