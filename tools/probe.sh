set -x
nproc; lscpu | grep -E "Model name|Socket|Core|Thread" ; free -g | head -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
CP=$!
./tools/fp64_peak
kill $CP
python -c "import mpmath; print('mpmath ok')"
