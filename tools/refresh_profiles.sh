# One gpurun call: C2 bench (own arm + reference arm), then the ncu launch list
# of the same bench command and an ncu --set full capture of one x-deferral
# cycle (8 PCG rounds) of the PCG kernels.  Usage: bash tools/refresh_profiles.sh [tag]
tag=${1:-r01}
set -x
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err || exit 1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python tools/rank_share.py --config c2 > gpurun_out/rank_share_c2.jsonl 2> gpurun_out/rank_share.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_spmm_ell|k_spmm_pq|k_update_r|k_update_p|k_update_xring" \
  -s 24 -c 24 -o gpurun_out/pcg_c2_$tag -f python tools/profile_pcg.py --config c2 --rounds 16 \
  > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
