# GPU session 46: per-launch tensor-core efficiency of the branchy models
for mdl in inception-v3 resnet-50 googlenet; do timeout 300 python tools/gemm_probe.py $mdl 30 > gpurun_out/gemm_probe_$mdl.txt 2>&1; done
head -5 gpurun_out/gemm_probe_*.txt
