timeout 1500 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/r02_gpuall.log 2>&1; tail -18 gpurun_out/r02_gpuall.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
