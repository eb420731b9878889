( time timeout 1700 python -m pytest tests/ -x -q -m gpu -n 0 --durations=15 ) > gpurun_out/gputest15_serial.log 2>&1; echo rc=$? >> gpurun_out/gputest15_serial.log
