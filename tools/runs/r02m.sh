cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ipsc.py -x -q > gpurun_out/r02m_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02m_pytest.log
