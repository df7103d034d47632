timeout 1500 bash tools/variants_run.sh cur lib:ct4 lib:ct8 lib:ct16 lib:ct8f lib:ct16f1 lib:ct32f1 lib:f2k lib:bc lib:bcct8 lib:bc2 lib:bc2ct8 cur > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log | cut -c1-150
