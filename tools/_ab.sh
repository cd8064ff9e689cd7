for i in 1 2; do
for lib in libffb200.so libffb200_old.so; do
  echo "== $lib"
  FFB200_LIB=paper_2505_22758_b200/$lib timeout 200 python tools/perf_probe.py --batch 16 --steps 20 2>&1 | grep fused_overlap
  FFB200_LIB=paper_2505_22758_b200/$lib timeout 200 python tools/perf_probe.py --batch 8 --steps 20 2>&1 | grep fused_overlap
done; done
