# prototype: v pass and merged x pass in v2 blocks on two streams (three buffers)
set -x
o=gpurun_out/r02b_ovl; mkdir -p $o
python scripts/proto_overlap.py --config small --blocks 1 4 --steps 5 > $o/small.json 2>&1
python scripts/proto_overlap.py --config cfg2 --blocks 1 2 4 8 16 --steps 20 > $o/cfg2.json 2>&1
python scripts/proto_overlap.py --config cfg2 --blocks 1 4 8 --steps 20 > $o/cfg2b.json 2>&1
python scripts/proto_overlap.py --config cfg3 --blocks 1 4 8 --steps 40 > $o/cfg3.json 2>&1
ls $o
