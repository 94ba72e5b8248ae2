# full GPU suite + smoke (round 2); parity numbers to gpurun_out/r2_parity.json
mkdir -p gpurun_out
python paper_2508_19737_b200/_build.py > gpurun_out/r2_build.log 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r2_smoke.log
IGP_PARITY_LOG=gpurun_out/r2_parity.json timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/r2_pytest_full.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/r2_pytest_full.log
