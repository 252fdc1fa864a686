set -x
mkdir -p gpurun_out/r02h
export DSGPU_TIMEOUT_S=60
python bench.py > gpurun_out/r02h/bench.json 2> gpurun_out/r02h/bench.err
tail -c 300 gpurun_out/r02h/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h/smoke.log 2>&1; tail -2 gpurun_out/r02h/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02h/bench_launches.csv python bench.py --no-cpu-baseline > gpurun_out/r02h/bench_under_ncu.log 2>&1
tail -c 200 gpurun_out/r02h/bench_under_ncu.log
DSGPU_TIMEOUT_S=100 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:minres_kernel -s 1 -c 1 --csv --log-file gpurun_out/r02h/traffic_c4.csv python tools/minres_profile.py c4 > gpurun_out/r02h/traffic_c4.log 2>&1
tail -3 gpurun_out/r02h/traffic_c4.csv | cut -c150-400
DSGPU_LIB_DIR=paper_1309_5048_b200/lib_diag timeout 300 python tools/phase_probe.py c4 2>/dev/null > gpurun_out/r02h/phases.jsonl
cat gpurun_out/r02h/phases.jsonl | cut -c1-1400
DSGPU_TIMEOUT_S=100 timeout 900 ncu --set full --clock-control none --import-source on -k regex:minres_kernel -s 1 -c 1 -o gpurun_out/r02h/minres_c4_full python tools/minres_profile.py c4 > gpurun_out/r02h/full_c4.log 2>&1
tail -3 gpurun_out/r02h/full_c4.log
