# e2e pipeline check + PCIe bound + fresh ncu of the dominant kernel (one GPU)
set -x
OUT=gpurun_out
timeout 120 python tools/pcie_probe.py > $OUT/pcie.json 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k async > $OUT/pytest_async.log 2>&1
timeout 300 python bench.py > $OUT/bench_default.json 2> $OUT/bench.err
bash tools/gpu_profile.sh
