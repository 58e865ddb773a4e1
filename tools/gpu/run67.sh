# GPU session 67: HEAD launch lists of the branchy models (Inception-v3, ResNet-50, GoogLeNet)
set -x
for mdl in inception-v3 resnet-50 googlenet; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches67_$mdl.csv python tools/model_launches.py $mdl 2 > gpurun_out/ncu67_$mdl.log 2>&1; echo $mdl rc $?
done
timeout 300 python tools/gemm_probe.py inception-v3 20 > gpurun_out/gemm_probe_inc67.txt 2>&1
