timeout 300 python tools/time_sweep.py --configs cfg2,cfg5 --stagings 0 --cycles 6 --lib _ab/prev/libmg.so > gpurun_out/sweep8.jsonl 2> gpurun_out/sweep8.err
timeout 300 python tools/time_sweep.py --configs cfg2,cfg5 --stagings 0 --cycles 6 >> gpurun_out/sweep8.jsonl 2>> gpurun_out/sweep8.err
timeout 120 python tools/time_sweep.py --configs cfg2 --stagings 1 --cycles 6 >> gpurun_out/sweep8.jsonl 2>> gpurun_out/sweep8.err
echo done >> gpurun_out/sweep8.err
