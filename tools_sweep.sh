cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools_legbench.py 2>&1 | tail -1
WL=aniso N=4095 timeout 120 python tools_legbench.py 2>&1 | tail -1
LEGS=down BMG_LIB=$PWD/variants_exp31.so timeout 60 python tools_legbench.py 2>&1 | tail -1
