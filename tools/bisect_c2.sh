# cfg2 solve time per library build (regression bisect)
# variants first: git worktree add /tmp/wt_C C; (cd /tmp/wt_C && SLSE_BUILD_OUT=$PWD/build/variants/bis_C python paper_1705_06073_b200/build.py)
for lib in build/variants/bis_72ec20e build/variants/bis_23aa0b4 build/variants/bis_7cbf127 paper_1705_06073_b200/_lib; do
  echo "== $lib"; for i in 1 2; do SLSE_LIB=$lib/libsuperlse_b200.so python tools/bench_configs.py --configs 2 --no-cpu; done
done
