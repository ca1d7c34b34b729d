set -u
o=gpurun_out/r2k; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1

timeout 300 python tools/tile_sweep.py > $o/sweep_tailsm.jsonl 2>> $o/sweep.err
BMG_TILE_POINTS=20000 N=255 WL=poisson NCYC=1 timeout 300 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_tile_down|k_tail" -c 3 -o $o/tile_full python tools/profile_cycle.py > $o/ncu.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_solve.py tests/test_gpu_pcg.py tests/test_gpu_block.py -m gpu -q -x > $o/tests.log 2>&1
