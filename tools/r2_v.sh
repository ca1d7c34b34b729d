set -u
o=gpurun_out/v; mkdir -p $o; rm -f $o/sweep.jsonl
for rep in 1 2; do VARIANTS="base rb" WLS="aniso:4095 poisson:8191" LEGS=down,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
cat $o/sweep.jsonl
BMG_LIB=$PWD/tools/vlib/libbmg_rb.so timeout 900 python -m pytest -q -x tests/test_gpu_fused_determinism.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py > $o/test_rb.log 2>&1; tail -1 $o/test_rb.log
