# GPU session 14: the rest of the single-GPU suite (continue after the fp32 tolerance fix) + branchy after the
# im2col/col2im rewrite + Inception launch list
set -x
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/t_full14.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py inception-v3 4 > gpurun_out/inc_plain14.log 2>&1; echo plain rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_inception14.csv python tools/model_launches.py inception-v3 2 > gpurun_out/ncu_inc14.log 2>&1; echo list rc $?
tail -5 gpurun_out/t_full14.log; tail -1 gpurun_out/inc_plain14.log
