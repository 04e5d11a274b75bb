for N in 512 1024 1536 2048 3072 4096; do python tools/pass_probe.py $N identity cfg3; done > gpurun_out/sweep.log 2>&1
SYLFEM_B200_PDL=0 python tools/pass_probe.py 2048 identity cfg3 >> gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
