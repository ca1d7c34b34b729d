set -u
o=gpurun_out/m; mkdir -p $o
for rep in 1 2; do VARIANTS="base merge" WLS="aniso:4095 poisson:8191" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
timeout 900 python -m pytest -q -x tests/test_gpu_fused_determinism.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fullcycle.py tests/test_gpu_dist.py tests/test_gpu_dist_shim.py > $o/test.log 2>&1; tail -1 $o/test.log
