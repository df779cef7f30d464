#!/bin/bash
# The SPEC's scaling experiments (acceptance 5-6) through the CLI on the B200
make -s -C tools/cli
C=tools/cli/spingp; O=gpurun_out/cli
$C scaling-n --method spingp,kf --ns 1000,2000,4000,8000 --out $O/n_spec 2> $O.n_spec.log
$C scaling-n --method spingp --ns 1000000,2000000,4000000,8000000 --out $O/n_gpu 2> $O.n_gpu.log
$C scaling-n --method dense --ns 200,400,800 --out $O/n_dense 2> $O.n_dense.log
$C scaling-b --method spingp,kf --bs 2,4,8,12,16 --n 1000 --out $O/b_spec 2> $O.b_spec.log
$C scaling-b --method spingp --bs 4,8,16 --n 1000000 --out $O/b_gpu 2> $O.b_gpu.log
