set -x
O=gpurun_out/diag2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
MPSW_PARITY_LOG=$O/parity.ndjson timeout 1200 python -m pytest tests/test_gpu_layers.py -q -rf --tb=short > $O/pytest_layers.txt 2>&1
for a in "opt-125m 1 8 31 --free" "opt-1.3b 1 8 31 --free"; do timeout 600 python tools/layer_parity.py $a >> $O/layers.ndjson 2>> $O/layers.err; done
