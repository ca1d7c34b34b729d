set -u
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullcycle.py tests/test_gpu_dist.py "tests/test_gpu_parity.py::test_random_shapes_vcycle_parity" -m gpu -q -s -rA > gpurun_out/r2b/fullcycle.log 2>&1
