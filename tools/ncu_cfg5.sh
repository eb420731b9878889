set -x
python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg5_s4.csv python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rb_pencil -c 1 -f -o gpurun_out/r02_s4_sweep4 python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/ncu_f1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rr2_pencil -c 1 -f -o gpurun_out/r02_s4_rr2_4 python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/ncu_f2.log 2>&1
ls -la gpurun_out/*.ncu-rep
