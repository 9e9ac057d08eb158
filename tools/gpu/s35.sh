timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/s35_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s35_smoke.txt 2>&1
timeout 2000 python bench.py > gpurun_out/s35_bench.json 2> gpurun_out/s35_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/s35_bench_ref.json 2> gpurun_out/s35_bench_ref.err
