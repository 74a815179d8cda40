#!/bin/bash
# End-of-round measurements on one B200 (run from the repo root under gpurun):
# bench lines for every workload, the reference arm, the ncu launch list of the
# default bench command, DRAM traffic captures and one ncu --set full of the
# headline kernel.  Outputs land in gpurun_out/ (copied to profiles/ by hand).
set -u
tag=${1:-r02}
mkdir -p gpurun_out
rm -f /dev/shm/mht_plans/c5* 2>/dev/null
for w in c2 c3 c1 c4 c2kd; do
  timeout 1500 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
  echo "bench $w rc=$?"; tail -c 300 gpurun_out/${tag}_bench_$w.json; echo
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference_c2.json 2>&1; echo "ref rc=$?"
# launch list of the default bench command (cold, serialised: compare shares)
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${tag}_c2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launch list rc=$?"
for w in c2 c3 c1 c4 c2kd; do
  timeout 600 python tools/prof_run.py $w > gpurun_out/${tag}_prof_$w.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_${w}_traffic.csv python tools/prof_run.py $w > gpurun_out/${tag}_ncu_traffic_$w.log 2>&1
  echo "traffic $w rc=$?"
done
# the c5 stand-in (103.6 GB plan, built by the device builder) last: the longest
if [ "${WITH_C5S:-0}" = "1" ]; then
  rm -f /dev/shm/mht_plans/*.plan 2>/dev/null  # host RAM: the 104 GB plan file lives in /dev/shm
  timeout 3000 python bench.py --workload c5s --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5s.json 2> gpurun_out/${tag}_bench_c5s.err
  echo "bench c5s rc=$?"; tail -c 300 gpurun_out/${tag}_bench_c5s.json; echo
fi
