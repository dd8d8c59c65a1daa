cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py > gpurun_out/r11_bench.json 2> gpurun_out/r11_bench.err; cat gpurun_out/r11_bench.json; tail -2 gpurun_out/r11_bench.err
python bench.py --impl reference > gpurun_out/r11_ref.json 2> gpurun_out/r11_ref.err; cat gpurun_out/r11_ref.json; tail -2 gpurun_out/r11_ref.err
