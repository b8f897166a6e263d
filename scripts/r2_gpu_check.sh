set -x
nproc; free -g | head -2; lscpu | grep 'Model name'
python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r2a_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench5.json 2> gpurun_out/r2a_bench5.err; echo "b5 rc=$?"
python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench4.json 2>&1; echo "b4 rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2a_ref.json 2>&1; echo "ref rc=$?"
cat gpurun_out/r2a_bench5.json gpurun_out/r2a_bench4.json gpurun_out/r2a_ref.json | cut -c1-2500
