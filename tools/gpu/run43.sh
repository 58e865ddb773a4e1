set -x
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_inception43.csv python tools/model_launches.py inception-v3 2 > gpurun_out/ncu_inc43.log 2>&1; echo list rc $?
