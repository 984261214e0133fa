#!/bin/bash
# Round evidence in one GPU call (run from the repo root on the GPU box):
#   bench lines, ncu launch lists of the bench command and of eager steps, ncu --set full
#   captures of the dominant kernels.  Everything lands in gpurun_out/; the summaries
#   worth keeping are copied into profiles/ afterwards.
set -u
O=gpurun_out
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/r02_bench_default.jsonl 2> $O/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/r02_bench_reference.jsonl 2> $O/bench_reference.err
for c in cfg1 cfg3 cfg4; do
  python bench.py --config $c --steps 10 --warmup 3 > $O/r02_bench_$c.json 2>> $O/bench_default.err
done
# launch lists of the bench command itself (per config; a number printed under ncu is not a bench value)
for c in cfg2 cfg5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file $O/r02_launches_bench_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline \
    > $O/ncu_bench_$c.log 2>&1
done
# eager steps (same kernels and shapes as the graphed bench)
for c in cfg2 cfg3 cfg5; do
  MPPS_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file $O/r02_launches_$c.csv python tools/one_step.py $c 3 > /dev/null 2>&1
done
# full captures of the dominant kernels (second launch of each: the paired power GEMM / Z^2)
MPPS_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz_gemm_pw16_kernel \
  --launch-skip 1 -c 1 -f -o $O/r02_ncu_cfg2_pw16 python tools/one_step.py cfg2 1 > $O/ncu_full_cfg2.log 2>&1
MPPS_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_gemm_wide_kernel \
  --launch-skip 1 -c 1 -f -o $O/r02_ncu_cfg5_wide python tools/one_step.py cfg5 1 > $O/ncu_full_cfg5.log 2>&1
# the headline's dominant launch itself: the paired [Z^3 | Z^4] product (N = 2n), third launch of the kernel
MPPS_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_gemm_wide_kernel \
  --launch-skip 2 -c 1 -f -o $O/r02_ncu_cfg5_wide_paired python tools/one_step.py cfg5 1 > $O/ncu_full_cfg5p.log 2>&1
MPPS_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz_gemm_pw16_kernel \
  --launch-skip 0 -c 1 -f -o $O/r02_ncu_cfg3_pw16 python tools/one_step.py cfg3 1 > $O/ncu_full_cfg3.log 2>&1
# text exports (the reports themselves exceed what gpurun copies back)
for r in r02_ncu_cfg2_pw16 r02_ncu_cfg5_wide r02_ncu_cfg5_wide_paired r02_ncu_cfg3_pw16; do
  if [ -f $O/$r.ncu-rep ]; then
    ncu -i $O/$r.ncu-rep --page details > $O/$r.txt 2>/dev/null
    ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
    ncu -i $O/$r.ncu-rep --page source --csv > $O/${r}_source.csv 2>/dev/null
    rm -f $O/$r.ncu-rep
  fi
done
ls -la $O | tail -30
