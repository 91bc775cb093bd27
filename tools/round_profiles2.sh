# Round-end evidence refresh: round_profiles.sh plus the superfast factor capture (N = 16384, 8 problems).
bash tools/round_profiles.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_dnc -c 1 -o gpurun_out/dnc_full -f \
  python tools/prof_factor.py --n 16384 --batch 8 --methods schur --reps 1 > gpurun_out/dnc_ncu.log 2>&1
