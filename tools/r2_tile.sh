set -u
o=gpurun_out/r2h; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
timeout 300 python tools/tile_sweep.py > $o/tile_sweep.jsonl 2> $o/tile_sweep.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_solve.py tests/test_gpu_pcg.py tests/test_gpu_fullcycle.py -m gpu -q -x > $o/tests.log 2>&1
