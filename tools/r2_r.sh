set -u
o=gpurun_out/r; mkdir -p $o
for rep in 1 2; do VARIANTS="base tst" WLS="checker:1023 poisson:8191" LEGS=cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
cat $o/sweep.jsonl
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullcycle.py tests/test_gpu_tail.py > $o/test.log 2>&1; tail -1 $o/test.log
