cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_f32tc.py -x -q -s 2>&1 | grep "f32tc n=\|passed\|failed\|Error\|error" | tail -30
