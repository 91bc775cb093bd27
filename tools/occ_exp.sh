# residency experiments: solver CTAs per SM x block size x shared region
# variants first: SLSE_BUILD_OUT=build/variants/mbwK SLSE_BUILD_DEFS=-DSLSE_SOLVER_MINB_WIDE=K python paper_1705_06073_b200/build.py (K = 2, 4)
A=build/variants/mbw2/libsuperlse_b200.so
B4=build/variants/mbw4/libsuperlse_b200.so
run() { c=$1; shift; echo "== cfg$c $*"; env "$@" timeout 600 python tools/bench_configs.py --configs $c --no-cpu; }
run 4 SLSE_LIB=$A SLSE_SOLVER_NT=256 SLSE_REGION_KB=110
run 4 SLSE_LIB=$B4 SLSE_SOLVER_NT=128 SLSE_REGION_KB=52
run 4 SLSE_LIB=$B4 SLSE_SOLVER_NT=128 SLSE_REGION_KB=36
run 3 X=1
run 3 SLSE_LIB=$A SLSE_SOLVER_NT=256 SLSE_REGION_KB=100
run 3 SLSE_LIB=$B4 SLSE_SOLVER_NT=128 SLSE_REGION_KB=52
run 5 SLSE_LIB=$A SLSE_SOLVER_NT=256 SLSE_REGION_KB=100
