for c in 2 3 4 5; do echo "== cfg$c"; SLSE_LIB=build/variants/prof/libsuperlse_b200.so timeout 300 python tools/solver_prof.py --config $c; done > gpurun_out/solver_prof.txt 2>&1
