set -u
o=gpurun_out/${TAG:-peer}; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x -k "bitwise" > $o/loop.log 2>&1; tail -2 $o/loop.log
timeout 900 python -m pytest tests/test_gpu_dist_shim.py -q -x -k "multi_rank and True" > $o/shim.log 2>&1; tail -3 $o/shim.log
