timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench10.json 2> gpurun_out/bench10.err
timeout 900 python tools/run_configs.py --json gpurun_out/configs10.jsonl > gpurun_out/configs10.log 2>&1
timeout 600 python tools/run_configs.py --only cfg2_m6,cfg3_m6,cfg4_m6,tube,tube_batched,tube_m6 --json gpurun_out/configs10.jsonl >> gpurun_out/configs10.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -n 8 > gpurun_out/gputest10.log 2>&1; echo rc=$? >> gpurun_out/gputest10.log
