set -x
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1
done
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
