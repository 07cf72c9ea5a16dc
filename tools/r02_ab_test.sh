#!/bin/bash
# fp32 tensor-core parity tests of the current build, then tools/r02_ab_multi.sh against ab/<names>
set -u
mkdir -p gpurun_out/abm
timeout 900 python -m pytest tests -m gpu -x -q -k "${AB_TESTS:-fp32tc or tensor_cores}" > gpurun_out/abm/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/abm/pytest.log
bash tools/r02_ab_multi.sh "$@"
