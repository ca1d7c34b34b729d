# Pairs-per-thread variants of the 9-point fused legs (tools/variants.py -> tools/vlib/):
# leg micro-benchmarks at 4095^2 anisotropic (9-point level 0) and 8191^2 Poisson cycles,
# then the fused-leg parity tests against each variant.
set -u
o=gpurun_out/ppt; mkdir -p $o
for rep in 1 2; do
  VARIANTS="${VARIANTS:-base p3 w128 u4}" WLS="${WLS:-aniso:4095 poisson:8191}" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err
done
for v in ${TESTV:-p3 w128 u4}; do
  BMG_LIB=$PWD/tools/vlib/libbmg_$v.so timeout 900 python -m pytest -q -x tests/test_gpu_fused_determinism.py tests/test_gpu_parity.py > $o/test_$v.log 2>&1
  tail -1 $o/test_$v.log
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
