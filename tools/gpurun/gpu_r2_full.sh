# full GPU test suite + smoke
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r2_full_pytest.txt
cat gpurun_out/r2_full_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
