# e2e (host-resident f) timeline at config 2 and block-count A/B in the bench
set -x
o=gpurun_out/r02b_e2e; mkdir -p $o
python scripts/e2e_timeline.py 16 > $o/timeline16.json 2>&1
python scripts/e2e_timeline.py 32 > $o/timeline32.json 2>&1
python scripts/pcie_probe.py > $o/pcie.json 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-blocks 16 > $o/b16.json 2> $o/b16.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-blocks 32 > $o/b32.json 2> $o/b32.err
ls $o
