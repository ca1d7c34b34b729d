# Programmatic dependent launch A/B (p0: BMG_PDL=0, p1: PDL on; tools/variants.py), then
# the GPU suite's cycle/solve/parity tests against p1.
set -u
o=gpurun_out/pdl; mkdir -p $o
for rep in 1 2; do
  VARIANTS="p0 p1" WLS="poisson:8191 aniso:4095 checker:1023 poisson:255" LEGS=cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err
done
BMG_LIB=$PWD/tools/vlib/libbmg_p1.so timeout 1500 python -m pytest -q -x tests/test_gpu_fused_determinism.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_solve.py tests/test_gpu_fullcycle.py tests/test_gpu_block.py tests/test_gpu_dist.py > $o/test_p1.log 2>&1
tail -1 $o/test_p1.log
