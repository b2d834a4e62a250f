#!/bin/bash
# The BASELINE.json configurations on one GPU (bench.py lines, one JSON per config) into $1 (a dir).
out=${1:-gpurun_out}
python bench.py --n-dims 6 --gaussians 4096 --batch 16384 --steps 20 --warmup 5 --no-secondary > $out/cfg1.json 2> $out/cfg1.err
python bench.py --impl reference --n-dims 6 --gaussians 4096 --batch 16384 --steps 3 --warmup 1 > $out/cfg1_ref.json 2> $out/cfg1_ref.err
python bench.py --children --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > $out/cfg2_children.json 2> $out/cfg2_children.err
python bench.py --n-dims 16 --gaussians 500000 --batch 4194304 --steps 2 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > $out/cfg4.json 2> $out/cfg4.err
python bench.py --n-dims 16 --gaussians 500000 --batch 4194304 --steps 2 --warmup 1 --regime C --no-secondary --no-e2e --no-cpu-baseline > $out/cfg4_C.json 2> $out/cfg4_C.err
python bench.py --gaussians 1000000 --batch 524288 --steps 3 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > $out/cfg5.json 2> $out/cfg5.err
python bench.py --gaussians 1000000 --batch 524288 --steps 3 --warmup 1 --regime C --children --no-secondary --no-e2e --no-cpu-baseline > $out/cfg5_C_children.json 2> $out/cfg5_C_children.err
python bench.py --gaussians 1000000 --batch 524288 --steps 3 --warmup 1 --regime G --no-secondary --no-e2e --no-cpu-baseline > $out/cfg5_G.json 2> $out/cfg5_G.err
