# x1 x x2 stencil passes: GPU tests (VirtualComm) and per-rank emulation of
# the 4 x 2 layout next to the x1-only and velocity-sharded layouts
set -x
o=gpurun_out/r02b_x2h; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q -p no:cacheprovider > $o/pytest_dist.log 2>&1; echo rc=$? >> $o/pytest_dist.log
python scripts/emulate_shards.py --config cfg2 --grid2d 4x2 --steps 5 > $o/emu_cfg2_4x2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg2 --grid2d 2x2 --steps 5 > $o/emu_cfg2_2x2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg3 --grid2d 4x2 --steps 5 > $o/emu_cfg3_4x2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg5 --grid2d 4x2 --steps 3 > $o/emu_cfg5_4x2.jsonl 2>&1
ls $o
