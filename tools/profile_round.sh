#!/bin/bash
# Round evidence, run on the GPU box (gpurun): bench lines (never under a profiler), the ncu launch
# list of the same command, one `ncu --set full` capture per hot kernel, the per-phase traces.
# usage: bash tools/profile_round.sh <tag>      outputs under gpurun_out/<tag>_*
set -u
tag=${1:-r02f}
out=gpurun_out
mkdir -p $out
python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
python bench.py --impl reference > $out/${tag}_bench_reference.json 2>> $out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-others --no-cpu-baseline > $out/${tag}_ncu_bench.log 2>&1
# the two kernels of a C5 step: 1024 matrices, second repetition (first = warm-up)
ncu --set full --clock-control none --import-source on -k regex:'pbtrf_cta_kernel|pbtrs_sweep_kernel' \
    --launch-skip 2 --launch-count 2 -f -o $out/${tag}_c5 python tools/prof_c5.py 1024 2 solve > $out/${tag}_ncu_c5.log 2>&1
# the whole-GPU kernel on C4 and C2 (second repetition)
ncu --set full --clock-control none --import-source on -k regex:band_multi_kernel --launch-skip 1 --launch-count 1 \
    -f -o $out/${tag}_c4 python tools/prof_one.py C4 2 > $out/${tag}_ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:band_multi_kernel --launch-skip 1 --launch-count 1 \
    -f -o $out/${tag}_c2 python tools/prof_one.py C2 2 > $out/${tag}_ncu_c2.log 2>&1
export BCG_LIB=$PWD/paper_2305_04635_b200/libbandchol_b200_trace.so
python tools/timing.py trace C2 C3 C4 > $out/${tag}_trace_multi.jsonl 2>&1
python tools/timing.py trace_la > $out/${tag}_trace_cta.jsonl 2>&1
python tools/timing.py trace_solve > $out/${tag}_trace_solve.jsonl 2>&1
unset BCG_LIB
python tools/timing.py rhs > $out/${tag}_rhs.jsonl 2>&1
./tools/micro/potrf_lab.bin > $out/${tag}_potrf_lab.txt 2>&1
ls -la $out | tail -20
