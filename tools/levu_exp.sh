# register Levinson: unrolled (120 instr/step, 30 KB body) vs compact rolled body, in warp mode
for lib in paper_1705_06073_b200/_lib/libsuperlse_b200.so build/variants/levu/libsuperlse_b200.so; do
  echo "== $lib"; for i in 1 2; do SLSE_LIB=$lib python tools/bench_configs.py --configs 1,2 --no-cpu; done
done
