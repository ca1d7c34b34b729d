set -u
o=gpurun_out/bb; mkdir -p $o; rm -f $o/sweep.jsonl
for rep in 1 2; do VARIANTS="k0 km6 k4" WLS="checker:1023 poisson:8191 aniso:4095 checker512:4095 poisson:2047 poisson:511" LEGS=cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
cat $o/sweep.jsonl
timeout 900 python -m pytest -q -x tests/test_gpu_fused_determinism.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py > $o/test.log 2>&1; tail -1 $o/test.log
