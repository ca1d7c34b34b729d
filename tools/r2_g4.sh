set -u
o=gpurun_out/r2f; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
VARIANTS="base g4" WLS="poisson:8191 aniso:4095" bash tools/sweep.sh > $o/sweep.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $o/parity.log 2>&1
for n in 8191 4095; do for wl in poisson aniso; do N=$n WL=$wl timeout 120 python tools/profile_setup.py >> $o/setup.log 2>&1; done; done
