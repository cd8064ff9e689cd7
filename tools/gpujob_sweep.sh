mkdir -p gpurun_out
timeout 1500 python tools/pipeline_sweep.py --measure --ctx 3072 --reps 2 --out gpurun_out/pipeline_sweep.json > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?"; tail -25 gpurun_out/sweep.log
timeout 600 python tools/pipeline_sweep.py --report --inp gpurun_out/pipeline_sweep.json --out gpurun_out/pipeline_sweep_report.json > gpurun_out/sweep_report.log 2>&1; echo "report rc=$?"; tail -40 gpurun_out/sweep_report.log
for tool in synccheck racecheck memcheck; do
  FFB200_LIB=$PWD/libffb200_san.so timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_toy.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -6 gpurun_out/san_$tool.log
done
