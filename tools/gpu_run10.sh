timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 bash tools/variants_run.sh cur lib:hb4 lib:hb4b3 lib:hb2b3 cur lib:hb4 lib:hb4b3 > gpurun_out/variants10.log 2>&1
cat gpurun_out/variants10.log | cut -c1-150
