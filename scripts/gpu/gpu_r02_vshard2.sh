# round 2: velocity-sharded dG with H = 1 and the boundary-first x pass (overlap)
set -x
o=gpurun_out/r02v2; mkdir -p $o
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -m gpu > $o/pytest_dist.log 2>&1
tail -3 $o/pytest_dist.log
python scripts/emulate_shards.py --config cfg2 --worlds 2 4 8 --steps 5 --vshard > $o/emu_cfg2_v.jsonl 2>&1
python scripts/emulate_shards.py --config cfg3 --worlds 2 4 8 --steps 10 --vshard > $o/emu_cfg3_v.jsonl 2>&1
python scripts/emulate_shards.py --config cfg5 --worlds 2 4 8 --steps 3 --vshard > $o/emu_cfg5_v.jsonl 2>&1
cat $o/*.jsonl | grep "{"
