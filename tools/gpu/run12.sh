# GPU session 12: branch-group tests (masked teacher-forced dgrad) + Inception-v3 launch list
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -s > gpurun_out/t_branchy.log 2>&1; echo branchy rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_inception.csv python tools/model_launches.py inception-v3 2 > gpurun_out/ncu_inc.log 2>&1; echo list rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain.log 2>&1; echo plain rc $?
tail -3 gpurun_out/t_branchy.log; cat gpurun_out/inc_plain.log | tail -2
