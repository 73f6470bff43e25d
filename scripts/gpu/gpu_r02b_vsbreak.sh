# where the emulated per-rank time of the velocity-sharded step goes
set -x
o=gpurun_out/r02b_vsb; mkdir -p $o
python scripts/vshard_breakdown.py --config cfg2 --world 8 --steps 5 > $o/cfg2_w8.json 2>&1
python scripts/vshard_breakdown.py --config cfg2 --world 4 --steps 5 > $o/cfg2_w4.json 2>&1
python scripts/vshard_breakdown.py --config cfg5 --world 8 --steps 3 > $o/cfg5_w8.json 2>&1
ls $o
