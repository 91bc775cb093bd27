# v5 grid kernel: timing (default + variants), parity, ncu capture
# variant first: SLSE_BUILD_OUT=build/variants/g5r112 SLSE_BUILD_DEFS=-DSLSE_G5_MAXREG=112 python paper_1705_06073_b200/build.py
python tools/grid_bench.py > gpurun_out/g5_bench.txt 2>&1
SLSE_LIB=build/variants/g5r112/libsuperlse_b200.so python tools/grid_bench.py >> gpurun_out/g5_bench.txt 2>&1
SLSE_GRID_V3=1 python tools/grid_bench.py >> gpurun_out/g5_bench.txt 2>&1
python -m pytest tests -m gpu -x -q -k "per_call" > gpurun_out/g5_pytest.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:grid_tma -c 1 -o gpurun_out/g5_full -f python tools/grid_bench.py --reps 1 > gpurun_out/g5_ncu.log 2>&1
