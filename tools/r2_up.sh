set -u
o=gpurun_out/r2m; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
VARIANTS="cur u128 u128p2 u256p1" WLS="poisson:8191" LEGS=up,cycle bash tools/sweep.sh > $o/sweep.jsonl 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_tile.py > $o/san_racecheck_tile.txt 2>&1
