( time timeout 1500 python -m pytest tests/ -x -q -m gpu ) > gpurun_out/gputest14_default.log 2>&1; echo rc=$? >> gpurun_out/gputest14_default.log
( time timeout 1700 python -m pytest tests/ -x -q -m gpu -n 0 --durations=30 ) > gpurun_out/gputest14_serial.log 2>&1; echo rc=$? >> gpurun_out/gputest14_serial.log
