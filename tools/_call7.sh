python tools/time_sweep.py --configs cfg2,cfg5 --stagings 0,1 --cycles 6 > gpurun_out/sweep7.jsonl 2> gpurun_out/sweep7.err
python tools/time_sweep.py --configs cfg2,cfg5 --stagings 0 --cycles 6 --lib _ab/prev/libmg.so >> gpurun_out/sweep7.jsonl 2>> gpurun_out/sweep7.err
timeout 900 python -m pytest tests -m gpu -x -q -n 8 -k "smooth or variants or vcycle or tma" > gpurun_out/gputest7.log 2>&1; echo rc=$? >> gpurun_out/gputest7.log
