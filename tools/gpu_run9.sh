HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_lean.so timeout 600 python -m pytest tests/test_gpu_solver.py tests/test_gpu_leadfield.py -x -q 2>&1 | tail -2
timeout 900 bash tools/variants_run.sh cur lib:lean cur lib:lean > gpurun_out/variants9.log 2>&1
cat gpurun_out/variants9.log | cut -c1-150
for b in 16 32; do echo "batch $b lean: $(HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_lean.so HFB200_MAX_BATCH=$b timeout 300 python tools/profile_pcg.py --config c2 --rounds 16 2>&1 | grep -o "'kernels'.*" | cut -c1-120)"; done
