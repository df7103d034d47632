HFB200_LIB=$PWD/paper_1811_07717_b200/_lib/variants/libhfb200_sm.so timeout 600 python -m pytest tests/test_gpu_solver.py -x -q 2>&1 | tail -3
timeout 900 bash tools/variants_run.sh cur lib:sm cur lib:sm > gpurun_out/variants5.log 2>&1
cat gpurun_out/variants5.log | cut -c1-150
timeout 600 python tools/rank_share.py --config c5 --n 8 --steps 2 > gpurun_out/rank_share_c5.jsonl 2> gpurun_out/rank_share_c5.err; tail -2 gpurun_out/rank_share_c5.err; cat gpurun_out/rank_share_c5.jsonl
