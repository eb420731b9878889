set -e
python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/plain6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rb_pencil -s 0 -c 1 -o gpurun_out/r02_sweep4 python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/ncu6a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rr2_pencil -s 0 -c 1 -o gpurun_out/r02_rr2_4 python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/ncu6b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_c2f_thin -s 3 -c 1 -o gpurun_out/r02_thin4 python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/ncu6c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5_v3.csv python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/ncu6d.log 2>&1
