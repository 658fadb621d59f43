set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest -x -q -m gpu tests/test_batch_gpu.py 2>&1 | tail -30
timeout 900 python -m pytest -x -q -m gpu tests/test_pipeline_gpu.py tests/test_layer_tree_gpu.py tests/test_plugin_gpu.py tests/test_captures.py 2>&1 | tail -5
