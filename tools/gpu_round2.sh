#!/bin/bash
# Round-2 check under gpurun: the GPU suite, smoke(), the default bench line
# (cfg5 headline) and the ncu launch list of a short bench (this library's kernels).
set -x
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_r02.log 2>&1; echo pytest_rc=$?
tail -20 gpurun_out/pytest_gpu_r02.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke_r02.log
timeout 1800 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo bench_rc=$?
tail -c 1500 gpurun_out/bench_r02.json
SYLFEM_B200_GRAPH=chunked ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --kernel-name-base demangled -k regex:"sfb::" --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 1 --warmup 1 --iters-per-step 3 --no-cpu-baseline --no-e2e --no-alt --no-secondary \
  > gpurun_out/ncu_launch_r02.log 2>&1; echo ncu_rc=$?
