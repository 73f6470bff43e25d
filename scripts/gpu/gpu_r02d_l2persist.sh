# fourth session: config 5 composed x pass with a persisting-L2 carve-out (density slabs, evict_last)
set -x
o=gpurun_out/r02d_l2persist; mkdir -p $o
for m in 0 64 0 64; do
python scripts/l2persist_probe.py $m --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $o/bench_cfg5_p${m}_$RANDOM.json 2>> $o/err_$m.log
done
ls -la $o
