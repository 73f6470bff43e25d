# emulated per-rank compute over the driver's step count (20; config 5: 10),
# so the opening / closing single x passes are amortized as in the 1-GPU line
set -x
o=gpurun_out/r02b_emu; mkdir -p $o
python scripts/emulate_shards.py --config cfg2 --worlds 2 4 8 --steps 20 --vshard > $o/cfg2_v2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg2 --grid2d 4x2 --steps 20 > $o/cfg2_4x2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg2 --worlds 8 --steps 20 > $o/cfg2_x1.jsonl 2>&1
python scripts/emulate_shards.py --config cfg3 --worlds 2 4 8 --steps 20 --vshard > $o/cfg3_v2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg5 --worlds 2 4 8 --steps 10 --vshard > $o/cfg5_v2.jsonl 2>&1
python scripts/vshard_breakdown.py --config cfg2 --world 8 --steps 20 > $o/cfg2_w8_break20.json 2>&1
ls $o
