# Group-wait variants (BMG_GWAIT 0/1/2, built by tools/variants.py into tools/vlib/):
# level-0 legs + cycle at 8191^2 Poisson (5-point) and 4095^2 anisotropic (9-point),
# then the fused-leg parity/determinism tests against each variant.
set -u
o=gpurun_out/gw; mkdir -p $o
for rep in 1 2; do
  VARIANTS="${VARIANTS:-g0 g1 g2}" WLS="poisson:8191 aniso:4095" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err
done
for v in ${TESTV:-g1 g2}; do
  BMG_LIB=$PWD/tools/vlib/libbmg_$v.so timeout 900 python -m pytest -q -x tests/test_gpu_fused_determinism.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py > $o/test_$v.log 2>&1
  tail -1 $o/test_$v.log
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
