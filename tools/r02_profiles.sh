#!/bin/bash
# Round-2 ncu evidence (run on the B200 box; outputs under gpurun_out/r02/).
#   1. launch list of the default bench command (cold-cache, serialised)
#   2. ncu --set full of the three per-slice kernels of C2 (mode 0, tail, insertion)
#   3. ncu --set full of the mode-0 projection at the C3 / C4 / C5 sizes and of
#      the growth kernels (Gram, tridiagonal eigensolve) on a C5 growth epoch
# Every profiled command is first run WITHOUT ncu and must exit 0.
set -u
out=gpurun_out/r02
mkdir -p $out
B="python bench.py --steps 12 --warmup 5 --no-cpu-baseline --e2e-steps 0"
$B > $out/bench_plain.json 2> $out/bench_plain.err || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $out/launches_c2.csv $B > $out/ncu_launches.log 2>&1
# steady-state slices only: skip init + priming (kernel-name filtered)
ncu --set full --clock-control none --import-source on \
    -k regex:"proj0_cols|proj0_tma|tail_kernel|isvd_clu|isvd_grid|isvd_cta" -s 60 -c 9 \
    -o $out/c2_full -f $B > $out/ncu_c2_full.log 2>&1
python tools/ncu_summary.py $out/c2_full_summary.csv $out/c2_full.ncu-rep > /dev/null 2>&1
ncu -i $out/c2_full.ncu-rep --page details > $out/c2_full_details.txt 2>&1
rm -f $out/c2_full.ncu-rep
# other configs: mode-0 projection kernels (whatever variant the engine picks)
for cfg in c5 c3; do
  C="python bench.py --config $cfg --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0"
  $C > $out/bench_${cfg}_plain.json 2> $out/bench_${cfg}_plain.err || { echo "$cfg plain failed"; continue; }
  ncu --set full --clock-control none --import-source on \
      -k regex:"proj0_cols|proj0_tma|proj_dmma|proj0_fma" -s 20 -c 3 \
      -o $out/${cfg}_mode0_full -f $C > $out/ncu_${cfg}_mode0.log 2>&1
  python tools/ncu_summary.py $out/${cfg}_mode0_summary.csv $out/${cfg}_mode0_full.ncu-rep > /dev/null 2>&1
  ncu -i $out/${cfg}_mode0_full.ncu-rep --page details > $out/${cfg}_mode0_details.txt 2>&1
  rm -f $out/${cfg}_mode0_full.ncu-rep
done
# growth kernels: Gram + tridiagonal eigensolve on a 384-row mode (C4's size)
G="python tools/eig_route_timing.py child"
$G > $out/eig_plain.txt 2>&1 || echo "eig child failed"
ncu --set full --clock-control none --import-source on \
    -k regex:"tridiag_coop|tri_bisect|tri_invit|tri_backtransform|gram_partial_dmma" -s 40 -c 10 \
    -o $out/growth_full -f $G > $out/ncu_growth.log 2>&1
python tools/ncu_summary.py $out/growth_summary.csv $out/growth_full.ncu-rep > /dev/null 2>&1
ncu -i $out/growth_full.ncu-rep --page details > $out/growth_details.txt 2>&1
rm -f $out/growth_full.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    -k regex:"tridiag_coop|tri_bisect|tri_invit|tri_backtransform|gram_|sym_eig" \
    --log-file $out/launches_growth.csv $G > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep; du -sh gpurun_out; ls -la $out
