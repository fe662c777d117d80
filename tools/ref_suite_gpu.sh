#!/bin/bash
# Run the REFERENCE's own pkg/tests against the drop-in on a GPU box:
# stage (here, where /root/reference exists) -> gpurun -> remove the stage.
# The staged copy is git-ignored and lives only for the duration of the call.
set -e
cd "$(dirname "$0")/.."
python tests/ref_suite/stage.py .refsuite > /dev/null
/usr/local/graft/bin/gpurun --timeout 1800 -- 'mkdir -p gpurun_out; cd .refsuite && PYTHONPATH=$PWD:$GRAFT_REPO_ROOT timeout 1500 python -m pytest tests -q -p no:cacheprovider -rfE > ../gpurun_out/r02_reference_suite.txt 2>&1; tail -3 ../gpurun_out/r02_reference_suite.txt' || true
rm -rf .refsuite
