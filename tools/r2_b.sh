# Tail kernel rewrite (2-D thread map, reciprocal plane) tests + configs 1/2, and the
# pairs-per-thread sweep of the 5-point / 9-point-up legs (tools/vlib variants).
set -u
o=gpurun_out/b; mkdir -p $o
timeout 900 python -m pytest -q -x tests/test_gpu_tail.py tests/test_gpu_parity.py tests/test_gpu_solve.py tests/test_gpu_fused_determinism.py > $o/test.log 2>&1; tail -1 $o/test.log
for c in poisson33 checker1025; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $o/bench_$c.json 2>$o/bench_$c.err; tail -c 300 $o/bench_$c.json
done
VARIANTS="base d5p4 d5p1 u9p1 p3e1" WLS="poisson:8191 aniso:4095" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err
VARIANTS="base d5p4 d5p1 u9p1 p3e1" WLS="poisson:8191 aniso:4095" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
