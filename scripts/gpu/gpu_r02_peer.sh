# round 2: velocity sharding with halos read in place from peer buffers
set -x
o=gpurun_out/r02p; mkdir -p $o
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_guards.py -q -m gpu > $o/pytest_dist.log 2>&1
tail -3 $o/pytest_dist.log; grep -E "FAIL|Error" $o/pytest_dist.log | head
