timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench16.json 2> gpurun_out/bench16.err
timeout 1200 python -m pytest tests/ -x -q -m gpu -n 8 > gpurun_out/gputest16.log 2>&1; echo rc=$? >> gpurun_out/gputest16.log
