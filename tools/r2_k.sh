set -u
o=gpurun_out/k; mkdir -p $o
for rep in 1 2; do VARIANTS="base e5u1 e5d1 e9u2 w5up256" WLS="poisson:8191 aniso:4095" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
