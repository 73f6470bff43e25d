# round 2: opt-in config 5 full-size parity (one step vs the reference on the host)
set -x
free -g
VPB_TEST_CFG5=1 timeout 2400 python -m pytest tests/test_gpu_parity_headline.py -q -s -m gpu -k config5 > gpurun_out/cfg5_parity.log 2>&1
tail -5 gpurun_out/cfg5_parity.log
