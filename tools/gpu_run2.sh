set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
python bench.py --steps 100 --warmup 10 --no-extras --no-cpu-baseline --batch 16 > gpurun_out/bench_b16.json 2> gpurun_out/bench_b16.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/traffic.sh 1 0.4; echo "traffic1 rc=$?"
bash tools/traffic.sh 16 0.4; echo "traffic16 rc=$?"
