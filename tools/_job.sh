export DSGPU_TIMEOUT_S=60
mkdir -p gpurun_out/r02i
timeout 300 python tools/config_probe.py c4 --modes=auto 2>/dev/null | cut -c560-800
DSGPU_BS_SMEM_WHOLE=1 timeout 300 python tools/config_probe.py c4 --modes=auto 2>/dev/null | cut -c560-800
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "blocked or emulated or world1 or two_handles" 2>&1 | tail -3
PROBE_MEMGUARD_GB=8 timeout 2400 python tools/config_probe.py c5 --modes=auto --ic0-gpu > gpurun_out/r02i/c5.jsonl 2> gpurun_out/r02i/c5.log
tail -3 gpurun_out/r02i/c5.log; cut -c1-1500 gpurun_out/r02i/c5.jsonl
