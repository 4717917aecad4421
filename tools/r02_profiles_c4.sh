#!/bin/bash
# ncu evidence for C4 (384^3 x 16, 7.25 GB slices): the mode-0 TTM, the residual Gram and the
# tridiagonal eigensolve of its growth path. Outputs under gpurun_out/r02/ (summaries only).
set -u
out=gpurun_out/r02
mkdir -p $out
C="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$C > $out/bench_c4_plain.json 2> $out/bench_c4_plain.err || { echo "c4 plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on \
    -k regex:"proj_dmma_kernel|proj0_cols|proj0_tma|gram_partial_dmma|tridiag_coop|tri_bisect" -s 8 -c 8 \
    -o $out/c4_full -f $C > $out/ncu_c4.log 2>&1
python tools/ncu_summary.py $out/c4_summary.csv $out/c4_full.ncu-rep > /dev/null 2>&1
ncu -i $out/c4_full.ncu-rep --page details > $out/c4_details.txt 2>&1
rm -f $out/c4_full.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 40 -c 400 \
    --log-file $out/launches_c4.csv $C > /dev/null 2>&1
python tools/ncu_tail.py $out/launches_c4.csv 0 | tail -40
cat $out/c4_summary.csv | cut -c1-330
