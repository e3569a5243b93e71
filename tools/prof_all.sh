set -x
mkdir -p gpurun_out/final
python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/final/gpu_tests.txt
python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 --no-cpu --no-pcg --no-cfg3 --no-callers > gpurun_out/final/launches.csv 2> gpurun_out/final/launches.err
python tools/launch_shares.py gpurun_out/final/launches.csv gpurun_out/final/launch_shares.txt gpurun_out/final/traffic.json > /dev/null 2>&1
for p in 4 6 8; do
  ncu --set full --import-source on --clock-control none -k regex:sf3_fast_kernel -s 2 -c 1 -o /tmp/k$p python tools/profile_apply.py --p $p --dofs 1e7 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/k$p.ncu-rep > gpurun_out/final/ncu_full_p$p.txt 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:block_ilu_packed -s 1 -c 1 -o /tmp/b4 python tools/bilu_prof.py 4 60 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/b4.ncu-rep > gpurun_out/final/ncu_bilu_packed_p4.txt 2>&1
python tools/vcycle_breakdown.py 4 116 > gpurun_out/final/vcycle_p4.txt 2>&1
python tools/vcycle_breakdown.py 7 66 > gpurun_out/final/vcycle_p7.txt 2>&1
python tools/gap_probe.py 2 3 4 5 6 7 8 > gpurun_out/final/gap_probe.txt 2>&1
ls -la gpurun_out/final
