for b in 64 32; do echo "c5 batch $b: $(HFB200_MAX_BATCH=$b timeout 600 python tools/profile_pcg.py --config c5 --rounds 16 2>&1 | grep -o "'pcg_round'.*" | cut -c1-520)"; done
