# GPU parity + per-config throughput + grid kernel + superfast factor phase clocks
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python tools/bench_configs.py --no-cpu > gpurun_out/configs.log 2>&1
python tools/grid_bench.py > gpurun_out/g5_bench.txt 2>&1
for n in 4096 16384; do SLSE_DNC_PROF=1 python tools/prof_factor.py --n $n --batch 64 --methods schur --reps 1; done > gpurun_out/dncprof.txt 2>&1
