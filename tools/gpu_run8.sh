timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_ell" -s 8 -c 1 -o gpurun_out/spmm_sm -f python tools/profile_pcg.py --config c2 --rounds 16 > gpurun_out/ncu_spmm.log 2>&1
tail -3 gpurun_out/ncu_spmm.log
