export DSGPU_TIMEOUT_S=30
for v in lib_k7 lib_k8 lib_k6; do
  echo "== $v"
  DSGPU_LIB_DIR=paper_1309_5048_b200/$v timeout 300 python tools/config_probe.py c4 --modes=auto 2>&1 | tail -1 | cut -c1-200
  DSGPU_LIB_DIR=paper_1309_5048_b200/$v timeout 300 python tools/config_probe.py c4 --modes=auto 2>/dev/null | cut -c540-700
done
