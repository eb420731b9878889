for lib in _ab/head/libmg.so _ab/thindiv/libmg.so; do
timeout 300 python tools/stage_breakdown.py --cfg cfg5 --cycles 5 --lib $lib >> gpurun_out/ab13.jsonl 2>> gpurun_out/ab13.err
done
