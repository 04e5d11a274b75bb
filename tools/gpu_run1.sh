set -x
free -g; nproc; nvidia-smi -L
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_a.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu_a.log
timeout 1800 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg5_a.json 2> gpurun_out/bench_cfg5_a.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_cfg5_a.json; tail -20 gpurun_out/bench_cfg5_a.err
