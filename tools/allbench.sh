#!/bin/bash
# every bench line of profiles/r2_bench_*.json, one GPU: bash tools/allbench.sh (JSON lines in gpurun_out/b/)
mkdir -p gpurun_out/b
run() { name=$1; shift; timeout 900 "$@" > gpurun_out/b/$name.json 2> gpurun_out/b/$name.err; echo "$name rc=$?"; }
run k2 python bench.py --steps 10 --warmup 3
run k2_ref python bench.py --impl reference --steps 5 --warmup 1
run k2_adoch python bench.py --solver adoch --steps 5 --warmup 3
run g1 python bench.py --config g1 --steps 5 --warmup 3
run t6 python bench.py --config t6 --steps 3 --warmup 2
run e7 python bench.py --config e7 --steps 3 --warmup 2
run e7_rowpart python bench.py --config e7 --rowpart --steps 3 --warmup 2
run r8 python bench.py --config r8 --steps 2 --warmup 1
run k2_gpus2 python bench.py --gpus 2 --steps 3 --warmup 3
