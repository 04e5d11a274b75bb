#!/bin/bash
# Round-2 (Strassen schedule) check under gpurun: the GPU suite, smoke(), the default
# bench line, the ncu launch list of a short bench, and ncu captures of the batched
# leaf GEMM and of the Strassen sum / assembly passes (DRAM traffic per launch).
set -x
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_r02b.log 2>&1; echo pytest_rc=$?
tail -20 gpurun_out/pytest_gpu_r02b.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke_r02b.log
timeout 1800 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo bench_rc=$?
tail -c 600 gpurun_out/bench_r02b.json
SYLFEM_B200_GRAPH=chunked ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --kernel-name-base demangled -k regex:"sfb::" --log-file gpurun_out/launches_r02b.csv \
  python bench.py --steps 1 --warmup 1 --iters-per-step 2 --no-cpu-baseline --no-e2e --no-alt --no-secondary --no-classic \
  > gpurun_out/ncu_launch_r02b.log 2>&1; echo ncu_rc=$?
python tools/batch_gemm_time.py 343 1024 343 512 49 512 > gpurun_out/batch_gemm_time.log 2>&1
python tools/strassen_probe.py 2047 4095 8192 > gpurun_out/strassen_probe.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"dgemm_nt" -s 3 -c 1 \
  -o gpurun_out/dgemm_batch343_full python tools/batch_gemm_time.py 343 1024 > gpurun_out/ncu_batch343.log 2>&1; echo ncu_full_rc=$?
STRASSEN_PROBE_LEVELS=3 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"strassen|dgemm_nt" -c 24 --csv --kernel-name-base demangled --log-file gpurun_out/strassen_passes.csv \
  python tools/strassen_probe.py 8192 > gpurun_out/ncu_strassen_passes.log 2>&1; echo ncu_passes_rc=$?
