# main-ring slack sweep of the 9-point down leg; tail tests; ncu capture of the tail kernel
set -u
o=gpurun_out/c; mkdir -p $o
timeout 600 python -m pytest -q -x tests/test_gpu_tail.py > $o/test.log 2>&1; tail -1 $o/test.log
for rep in 1 2; do
VARIANTS="base p3e2 p3e3 p2e1" WLS="aniso:4095 poisson:8191" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_tail_sm -s 3 -c 1 -o $o/tail33 python bench.py --config poisson33 --steps 3 --warmup 3 --no-cpu-baseline > $o/ncu.log 2>&1; tail -2 $o/ncu.log
