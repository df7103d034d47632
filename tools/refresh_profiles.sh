# Round profiles, two gpurun calls (each within ~30 min):
#   bash tools/refresh_profiles.sh bench [tag]   benches: C2 (own arm + reference arm), C3, C5, C4 EIT, rank shares
#   bash tools/refresh_profiles.sh ncu [tag]     ncu launch lists of one step (C2, C3, C4, C5) and --set full captures
what=${1:-bench}
tag=${2:-r02}
o=gpurun_out
set -x
if [ "$what" = bench ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > $o/${tag}_bench_c2.json 2> $o/${tag}_bench_c2.err
  timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > $o/${tag}_bench_c2_reference.json 2> $o/${tag}_bench_c2_reference.err
  timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > $o/${tag}_bench_c3.json 2> $o/${tag}_bench_c3.err
  timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $o/${tag}_bench_c5.json 2> $o/${tag}_bench_c5.err
  timeout 600 python tools/eit_c4.py > $o/${tag}_c4_eit.log 2>&1
  timeout 600 python tools/rank_share.py --config c2 > $o/${tag}_c2_rank_share.jsonl 2> $o/${tag}_rank_share.err
  timeout 600 python tools/rank_share.py --config c5 --n 8 > $o/${tag}_c5_rank_share.jsonl 2>> $o/${tag}_rank_share.err
else
  # everything is summarised here and the raw captures deleted: gpurun brings back <= 64 MiB
  for cfg in c2 c3 c4; do
    timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $o/${tag}_${cfg}_launches.csv python tools/one_step.py --config $cfg > $o/${tag}_ncu_launch_$cfg.log 2>&1
    python tools/launch_shares.py $o/${tag}_${cfg}_launches.csv $o/${tag}_${cfg}_launch_shares.csv \
      "one full $cfg step (tools/one_step.py --config $cfg between cudaProfilerStart/Stop)"
    rm -f $o/${tag}_${cfg}_launches.csv
  done
  # one x-deferral cycle (8 rounds) of the PCG kernels at C2 kp=64 and C5 kp=32
  for cfg in c2 c5; do
    timeout 900 ncu --set full --clock-control none \
      -k regex:"k_spmm|k_update_r|k_update_p|k_update_xring" -s 24 -c 24 -o $o/${tag}_pcg_$cfg -f \
      python tools/profile_pcg.py --config $cfg --rounds 16 > $o/${tag}_ncu_pcg_$cfg.log 2>&1
    python tools/ncu_summary.py $o/${tag}_pcg_$cfg.ncu-rep > $o/${tag}_pcg_${cfg}_ncu_full_summary.jsonl
  done
  python tools/make_traffic.py c2=$o/${tag}_pcg_c2.ncu-rep c5=$o/${tag}_pcg_c5.ncu-rep > $o/${tag}_traffic.log 2>&1
  cp profiles/traffic.json $o/${tag}_traffic.json
  rm -f $o/${tag}_pcg_c5.ncu-rep
  # the SpMM alone with source lines (kept: one kernel)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmm" -s 2 -c 1 \
    -o $o/${tag}_spmm64 -f python tools/pcg_round_probe.py > $o/${tag}_ncu_spmm.log 2>&1
  python tools/ncu_summary.py $o/${tag}_spmm64.ncu-rep > $o/${tag}_spmm64_ncu_full_summary.jsonl
  rm -f $o/${tag}_pcg_c2.ncu-rep
  # the LF tail, assembly and topology kernels of one C2 build
  timeout 900 ncu --set full --clock-control none --profile-from-start off \
    -k regex:"k_lf_tile|k_bt_t|k_blocks|k_row_fill|k_row_count|k_ell_fill|k_init|k_whitney|k_boundary" \
    -c 12 -o $o/${tag}_tail_asm_c2 -f python tools/one_step.py --config c2 > $o/${tag}_ncu_tail.log 2>&1
  python tools/ncu_summary.py $o/${tag}_tail_asm_c2.ncu-rep > $o/${tag}_tail_asm_c2_ncu_full_summary.jsonl
  rm -f $o/${tag}_tail_asm_c2.ncu-rep
  timeout 600 ncu --set full --clock-control none -k regex:"k_eit_sens|k_dof_blocks" -c 2 \
    -o $o/${tag}_eit_sens -f python tools/eit_sens_probe.py --reps 1 > $o/${tag}_ncu_eit.log 2>&1
  python tools/ncu_summary.py $o/${tag}_eit_sens.ncu-rep > $o/${tag}_eit_sens_ncu_full_summary.jsonl
  rm -f $o/${tag}_eit_sens.ncu-rep
  timeout 600 ncu --set full --clock-control none --profile-from-start off \
    -k regex:"k_meg_rhs|k_meg_primary|k_meg_elem" -c 3 -o $o/${tag}_meg -f python tools/one_step.py --config c3 \
    > $o/${tag}_ncu_meg.log 2>&1
  python tools/ncu_summary.py $o/${tag}_meg.ncu-rep > $o/${tag}_meg_ncu_full_summary.jsonl
  rm -f $o/${tag}_meg.ncu-rep
  du -sh $o
fi
