timeout 900 python -m pytest tests/ -x -q -m gpu -n 8 -k "pruned or coarse or vcycle or fullsize or tube" > gpurun_out/gputest18.log 2>&1; echo rc=$? >> gpurun_out/gputest18.log
for cfg in cfg4 cfg5; do
timeout 300 python tools/stage_breakdown.py --cfg $cfg --cycles 5 >> gpurun_out/ab18.jsonl 2>> gpurun_out/ab18.err
timeout 300 python tools/stage_breakdown.py --cfg $cfg --cycles 5 --extra '{"coarse_pruning": 2}' >> gpurun_out/ab18.jsonl 2>> gpurun_out/ab18.err
done
