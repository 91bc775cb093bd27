# register block Schur-Levinson: cfg3, cfg4 (superfast vs Levinson), standalone factor
python tools/bench_configs.py --configs 3 --no-cpu
python tools/bench_configs.py --configs 4 --no-cpu
SLSE_DNC_MIN=100000 python tools/bench_configs.py --configs 4 --no-cpu
SLSE_DNC_MIN=100000 SLSE_NO_PAIR=1 python tools/bench_configs.py --configs 4 --no-cpu
python tools/prof_factor.py --n 1024 --batch 148 --methods levinson,schur --reps 2
python tools/prof_factor.py --n 4096 --batch 148 --methods levinson,schur --reps 2
