for v in 0 1 2; do echo "variant $v"; SDB_K9_VARIANT=$v PYTHONPATH=. python scripts/convout_probe.py; done
python -m pytest tests/test_kernels_gpu.py -q -x -k conv_out 2>&1 | tail -2
