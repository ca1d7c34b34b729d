set -u
o=gpurun_out/r2e; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist_shim.py -m gpu -q -rA > $o/shim.log 2>&1
VARIANTS="base w32 w100 w300" WLS="poisson:8191 aniso:4095" bash tools/sweep.sh > $o/sweep.jsonl 2>&1
