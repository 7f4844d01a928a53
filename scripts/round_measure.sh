# Round-end measurement on a B200 box (run through gpurun): the GPU test suite,
# smoke(), the bench line and the reference arm, the ncu launch list of a short
# bench run. Outputs land in gpurun_out/.
set -x
python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
SECONDS=0; python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo bench rc=$? wall=${SECONDS}s
SECONDS=0; python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err; echo ref rc=$? wall=${SECONDS}s
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --cpu-sample 1000000 --pf-iterations 0 --no-extra > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
