set -x
mkdir -p gpurun_out/r02j
export DSGPU_TIMEOUT_S=60
python bench.py --impl reference > gpurun_out/r02j/bench_reference.json 2> gpurun_out/r02j/bench_reference.err
python bench.py > gpurun_out/r02j/bench.json 2> gpurun_out/r02j/bench.err
tail -c 300 gpurun_out/r02j/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j/smoke.log 2>&1; tail -2 gpurun_out/r02j/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02j/bench_launches.csv python bench.py --no-cpu-baseline > gpurun_out/r02j/bench_under_ncu.log 2>&1
DSGPU_TIMEOUT_S=100 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:minres_kernel -s 1 -c 1 --csv --log-file gpurun_out/r02j/traffic_c4.csv python tools/minres_profile.py c4 > gpurun_out/r02j/traffic_c4.log 2>&1
DSGPU_TIMEOUT_S=100 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:minres_kernel -s 2 -c 2 --csv --log-file gpurun_out/r02j/traffic_c2.csv python tools/minres_profile.py c2 > gpurun_out/r02j/traffic_c2.log 2>&1
DSGPU_LIB_DIR=paper_1309_5048_b200/lib_diag timeout 300 python tools/phase_probe.py c4 2>/dev/null > gpurun_out/r02j/phases.jsonl
DSGPU_TIMEOUT_S=100 timeout 900 ncu --set full --clock-control none --import-source on -k regex:minres_kernel -s 1 -c 1 -o gpurun_out/r02j/minres_c4_full python tools/minres_profile.py c4 > gpurun_out/r02j/full_c4.log 2>&1
tail -3 gpurun_out/r02j/full_c4.log
PROBE_MEMGUARD_GB=8 timeout 2400 python tools/config_probe.py c5 --modes=auto --ic0-gpu > gpurun_out/r02j/c5.jsonl 2> gpurun_out/r02j/c5.log
tail -3 gpurun_out/r02j/c5.log; cut -c1-300 gpurun_out/r02j/c5.jsonl
