# warp-mode rendezvous variants (groups per CTA, Levinson yield slices): cfg2 solve time
# variants first: SLSE_BUILD_OUT=build/variants/gN SLSE_BUILD_DEFS=-DSLSE_RV_GROUPS=N python paper_1705_06073_b200/build.py (N = 1, 2)
for lib in ${RV_LIBS:-paper_1705_06073_b200/_lib build/variants/g2 build/variants/g1}; do
  echo "== $lib"; for i in 1 2; do SLSE_LIB=$lib/libsuperlse_b200.so python tools/bench_configs.py --configs 2 --no-cpu; done
done
