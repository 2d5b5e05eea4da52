mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_cpp_dropin.py tests/test_noise.py -m gpu -q -p no:cacheprovider > gpurun_out/r02f/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --dist-selftest --no-extras --steps 5 > gpurun_out/r02f/selftest.json 2> gpurun_out/r02f/selftest.err; echo selftest=$?
timeout 600 python bench.py --dist-selftest --layout replicated --no-extras --steps 5 > gpurun_out/r02f/selftest_rep.json 2> gpurun_out/r02f/selftest_rep.err; echo selftest_rep=$?
