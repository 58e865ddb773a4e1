# GPU session 8: ResNet-50 after the per-channel-group BN / vectorised pool kernels
set -x
timeout 300 python tools/resnet_launches.py 4 > gpurun_out/resnet_plain8.log 2>&1; echo plain rc $?
timeout 900 python -m pytest tests/test_resnet_gpu.py -q -s -x > gpurun_out/t_resnet8.log 2>&1; echo resnet rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_resnet8.csv python tools/resnet_launches.py 2 > gpurun_out/ncu_resnet8.log 2>&1; echo list rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-fp32 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo bench rc $?
cat gpurun_out/resnet_plain8.log; tail -3 gpurun_out/t_resnet8.log
