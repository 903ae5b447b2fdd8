timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/full_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/full_tests.log 2>&1
tail -3 gpurun_out/full_tests.log
