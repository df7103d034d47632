timeout 900 python tools/eit_c4.py > gpurun_out/eit_c4.log 2>&1; tail -12 gpurun_out/eit_c4.log
for b in 64 128 32; do echo "batch $b: $(HFB200_MAX_BATCH=$b timeout 300 python tools/profile_pcg.py --config c2 --rounds 16 2>&1 | grep -o "'pcg_round'.*" | cut -c1-400)"; done
