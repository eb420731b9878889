for pb in 1 2 4; do
timeout 300 python tools/time_sweep.py --configs cfg5 --stagings 0 --cycles 6 --extra "{\"pencil_blocks\": $pb}" >> gpurun_out/sweep9.jsonl 2>> gpurun_out/sweep9.err
done
timeout 300 python tools/time_sweep.py --configs cfg5 --stagings 0 --cycles 6 --extra "{\"zsplit\": 2, \"pencil_blocks\": 1}" >> gpurun_out/sweep9.jsonl 2>> gpurun_out/sweep9.err
timeout 300 python tools/stage_breakdown.py --cfg cfg5 --cycles 5 --extra '{"pencil_blocks": 1}' >> gpurun_out/sb9.jsonl 2>> gpurun_out/sweep9.err
timeout 300 python tools/stage_breakdown.py --cfg cfg5 --cycles 5 --extra '{"pencil_blocks": 4}' >> gpurun_out/sb9.jsonl 2>> gpurun_out/sweep9.err
