# Round-end measurement on a B200 box (run through gpurun): the GPU test suite,
# smoke(), the bench line and the reference arm. Outputs land in gpurun_out/.
set -x
python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err; echo ref rc=$?
