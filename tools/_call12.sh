for lib in _ab/head/libmg.so _ab/fldg/libmg.so; do
timeout 300 python tools/time_sweep.py --configs cfg2,cfg5 --stagings 0 --cycles 6 --lib $lib >> gpurun_out/sweep12.jsonl 2>> gpurun_out/sweep12.err
done
