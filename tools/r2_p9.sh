set -u
o=gpurun_out/r2l; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
VARIANTS="g4 p9" WLS="poisson:8191 aniso:4095" bash tools/sweep.sh > $o/sweep.jsonl 2>&1
VARIANTS="g4 p9" WLS="aniso:4095" bash tools/sweep.sh >> $o/sweep.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pcg.py -m gpu -q -x > $o/tests.log 2>&1
compute-sanitizer --tool memcheck python tools/sanitize_fused.py > $o/san_memcheck.txt 2>&1
compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_fused.py > $o/san_racecheck.txt 2>&1
compute-sanitizer --tool synccheck python tools/sanitize_fused.py > $o/san_synccheck.txt 2>&1
