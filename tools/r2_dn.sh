set -u
o=gpurun_out/r2o; mkdir -p $o
VARIANTS="cur d192p3 d256p4 d128p2" WLS="poisson:8191" LEGS=down,cycle bash tools/sweep.sh > $o/sweep.jsonl 2>&1
VARIANTS="cur d192p3 d256p4" WLS="poisson:8191" LEGS=down,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>&1
