# Leg micro-benchmarks of libbmg variants built by tools/variants.py (run under gpurun):
# VARIANTS="base h100" [WLS="poisson:8191 aniso:4095"] bash tools/sweep.sh
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-h0 h1 h2}; do
  for w in ${WLS:-poisson:8191 aniso:4095}; do
    BMG_LIB=tools/vlib/libbmg_$v.so WL=${w%%:*} N=${w##*:} timeout 120 python tools/legbench.py
  done
done
