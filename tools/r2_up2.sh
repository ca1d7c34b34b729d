set -u
o=gpurun_out/r2n; mkdir -p $o
VARIANTS="cur u128p2 u64 u256p4 u192p3" WLS="poisson:8191" LEGS=up,cycle bash tools/sweep.sh > $o/sweep.jsonl 2>&1
VARIANTS="cur u128p2" WLS="poisson:8191" LEGS=up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>&1
