# one-warp FFT radix-8 passes vs radix-4 (solver GS apply / grid): cfg1-3 solve times
for lib in paper_1705_06073_b200/_lib/libsuperlse_b200.so build/variants/r8/libsuperlse_b200.so; do
  echo "== $lib"; SLSE_LIB=$lib python tools/bench_configs.py --configs 2,3 --no-cpu; SLSE_LIB=$lib python tools/bench_configs.py --configs 2 --no-cpu
done
