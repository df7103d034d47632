HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_opt5.so timeout 600 python -m pytest tests/test_gpu_solver.py tests/test_gpu_leadfield.py -x -q 2>&1 | tail -2
timeout 900 bash tools/variants_run.sh cur lib:opt5 lib:opt7 lib:opt4 cur lib:opt5 lib:opt7 lib:opt4 > gpurun_out/variants12.log 2>&1
cat gpurun_out/variants12.log | cut -c1-110
