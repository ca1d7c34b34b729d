set -u
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/gputest.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
nvidia-smi -q | grep -i -A3 "Clocks" | head -20 > gpurun_out/r2a/smi.txt
nproc > gpurun_out/r2a/nproc.txt; free -g >> gpurun_out/r2a/nproc.txt
