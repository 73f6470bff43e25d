# velocity-sharded merged x pass with one accumulating density per shard
# (vpb_dg_sweep_xcomp_rows): dist tests, emulation and breakdown at 20 steps
set -x
o=gpurun_out/r02b_xr; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q -p no:cacheprovider > $o/pytest_dist.log 2>&1; echo rc=$? >> $o/pytest_dist.log
python scripts/emulate_shards.py --config cfg2 --worlds 2 4 8 --steps 20 --vshard > $o/cfg2_v2.jsonl 2>&1
python scripts/vshard_breakdown.py --config cfg2 --world 8 --steps 20 > $o/cfg2_w8_break20.json 2>&1
python scripts/emulate_shards.py --config cfg3 --worlds 8 --steps 20 --vshard > $o/cfg3_v2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg5 --worlds 8 --steps 10 --vshard > $o/cfg5_v2.jsonl 2>&1
ls $o
