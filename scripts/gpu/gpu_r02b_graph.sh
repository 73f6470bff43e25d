# AdvanceGraph tests and bench lines with the K-step block replayed from a CUDA graph
set -x
o=gpurun_out/r02b_graph; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -x -q -p no:cacheprovider -k "graph" > $o/pytest_graph.log 2>&1; echo rc=$? >> $o/pytest_graph.log
python bench.py --config cfg1 --no-cpu-baseline --graph > $o/cfg1_graph.json 2> $o/cfg1_graph.err
python bench.py --config cfg1 --no-cpu-baseline > $o/cfg1_eager.json 2> $o/cfg1_eager.err
python bench.py --config cfg3 --no-cpu-baseline --no-e2e --graph > $o/cfg3_graph.json 2> $o/cfg3_graph.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graph > $o/cfg2_graph.json 2> $o/cfg2_graph.err
ls $o
