set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python tools/meshgen_bench.py > gpurun_out/meshgen_bench.jsonl 2> gpurun_out/meshgen_bench.err; tail -3 gpurun_out/meshgen_bench.err
cat gpurun_out/meshgen_bench.jsonl
timeout 600 python tools/rank_share.py --config c2 > gpurun_out/rank_share_c2.jsonl 2> gpurun_out/rank_share.err; tail -2 gpurun_out/rank_share.err
cat gpurun_out/rank_share_c2.jsonl
timeout 900 bash tools/variants_run.sh cur lib:ct4 lib:ct8 lib:ct16 lib:ct8f lib:ct16f1 lib:ct32f1 lib:f2k > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log
