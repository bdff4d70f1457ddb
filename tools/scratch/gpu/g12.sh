mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/g12_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/g12_tests.txt
timeout 900 python tools/run_reference_suite.py -q -rf --tb=line > gpurun_out/g12_refsuite.txt 2>&1
echo "rc=$?" >> gpurun_out/g12_refsuite.txt
timeout 1500 python bench.py > gpurun_out/g12_bench.json 2> gpurun_out/g12_bench.err
echo "rc=$?" >> gpurun_out/g12_bench.err
