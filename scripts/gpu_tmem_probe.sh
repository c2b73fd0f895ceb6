# TMEM <-> register throughput probe (scripts/probes/tmem_bw.cu)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/tmem_bw scripts/probes/tmem_bw.cu && timeout 120 gpurun_out/tmem_bw > gpurun_out/tmem_bw.txt 2>&1
rm -f gpurun_out/tmem_bw
