cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-h0 h1 h2}; do
  BMG_LIB=variants/libbmg_$v.so timeout 120 python tools/legbench.py
  BMG_LIB=variants/libbmg_$v.so WL=aniso N=4095 timeout 120 python tools/legbench.py
done
