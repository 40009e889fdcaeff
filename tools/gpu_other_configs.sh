# bench lines for the other BASELINE configs at HEAD
set -x
mkdir -p gpurun_out
for c in c2 c4a c4b; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c $?"
done
