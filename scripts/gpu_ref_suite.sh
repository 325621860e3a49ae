#!/bin/bash
# the reference's own pytest suite, every Context replaced by the GPU context
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
cd baseline/_ref/cryptogen_tests && PYTHONPATH=$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT:$GRAFT_REPO_ROOT/scripts \
  timeout ${T:-2400} python -m pytest -p ref_suite_plugin -q ${ARGS:-.} 2>&1 | tail -150 > $GRAFT_REPO_ROOT/gpurun_out/ref_suite.log
tail -15 $GRAFT_REPO_ROOT/gpurun_out/ref_suite.log
