set -u
o=gpurun_out/aa; mkdir -p $o; rm -f $o/sweep.jsonl
for rep in 1 2; do VARIANTS="base w128p2 w128p1" WLS="poisson:8191" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
cat $o/sweep.jsonl; tail -3 $o/sweep.err
