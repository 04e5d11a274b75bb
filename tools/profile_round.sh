#!/bin/bash
# Round profiling recipe (run under gpurun from the repo root): the default
# bench line, the ncu launch list of a short bench, and full captures of the
# MO-PCG passes (DRAM traffic for bench's roofline_hbm.traffic).
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
# (only this library's kernels: bench.py also times cuBLAS for the roofline peak)
SYLFEM_B200_GRAPH=chunked ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --kernel-name-base demangled -k regex:"sfb::" \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --iters-per-step 10 --no-full \
  --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"band_kernel" -s 6 -c 1 \
  -o gpurun_out/band_full python tools/pass_probe.py 2048 identity cfg3 > gpurun_out/ncu_band.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"pcg_rupdate" -s 6 -c 1 \
  -o gpurun_out/rupdate_full python tools/pass_probe.py 2048 identity cfg3 > gpurun_out/ncu_rupdate.log 2>&1
tail -2 gpurun_out/bench.err
