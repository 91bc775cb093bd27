set -x
mkdir -p gpurun_out
python tools/grid_omega_bench.py --probe --old --shapes 256:1024:10752,256:1024:43008 > gpurun_out/gc_main.txt 2>&1
for v in gc2 gc4; do echo "== $v" >> gpurun_out/gc_main.txt; SLSE_LIB=build/variants/$v/libsuperlse_b200.so python tools/grid_omega_bench.py --shapes 256:1024:43008 >> gpurun_out/gc_main.txt 2>&1; done
python tools/grid_omega_bench.py --old --shapes 64:256:43008,1024:4096:10752,4096:16384:2688,16384:65536:672 >> gpurun_out/gc_main.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "grid_eval" > gpurun_out/gc_tests.txt 2>&1
tail -3 gpurun_out/gc_tests.txt
cat gpurun_out/gc_main.txt
