timeout 600 python tools/e2e_init_breakdown.py 2>&1 | tail -3
for b in 16 32; do echo "batch $b: $(HFB200_MAX_BATCH=$b timeout 300 python tools/profile_pcg.py --config c2 --rounds 16 2>&1 | grep -o "'pcg_round'.*" | cut -c1-500)"; done
