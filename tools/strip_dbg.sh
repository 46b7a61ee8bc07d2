timeout 600 python -m pytest tests/test_parity.py -m gpu -q -x -k "strips_emulated" 2>&1 | grep -E "Error|error|assert|mismatch" | head -20 > gpurun_out/strip_dbg.log
