# GPU session 7: ResNet-50 step launch list, resnet tests, headline parity (full)
set -x
timeout 300 python tools/resnet_launches.py 2 > gpurun_out/resnet_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_resnet.csv python tools/resnet_launches.py 2 > gpurun_out/ncu_resnet.log 2>&1; echo list rc $?
timeout 900 python -m pytest tests/test_resnet_gpu.py -q -s > gpurun_out/t_resnet.log 2>&1; echo resnet rc $?
timeout 1200 python -m pytest tests/test_headline_parity_gpu.py -q -s > gpurun_out/t_headline.log 2>&1; echo headline rc $?
cat gpurun_out/resnet_plain.log
