# GPU session 50: the flat (GEMM-engine) conv backward-filter at narrow channels (Inception's stem)
set -x
for sh in 147,32,32 147,32,64 73,96,192 35,64,96; do timeout 120 python tools/probe_conv.py --shape $sh --iters 10; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100_kernel -s 1 -c 1 -o gpurun_out/prof_wgrad_flat_32 python tools/probe_conv.py --shape 147,32,32 --op wgrad --iters 1 > gpurun_out/ncu_wg32.log 2>&1; echo cap rc $?
