# Superfast-leaf A/B: standalone factor times (N = 16384 / 4096), cfg3-5 solve times, GPU parity subset.
python tools/prof_factor.py --n 16384 --batch 8 --methods schur --reps 2 > gpurun_out/pf.txt 2>&1
python tools/prof_factor.py --n 4096 --batch 148 --methods schur --reps 2 >> gpurun_out/pf.txt 2>&1
python tools/bench_configs.py --no-cpu --configs ${CFGS:-4,5} > gpurun_out/configs.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
cat gpurun_out/pf.txt gpurun_out/configs.log; tail -3 gpurun_out/gputest.log
