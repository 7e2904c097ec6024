# The reference's own test suite (baseline/_ref/tests, copied from
# /root/reference/pkg/tests) against the GPU drop-in through the import shim.
export PYTHONPATH=tools/refshim:baseline/_ref/tests
mkdir -p gpurun_out
python -m pytest -p refshim_plugin baseline/_ref/tests -q -p no:cacheprovider -rfE --durations=15 \
  > gpurun_out/reference_suite.log 2>&1
echo "reference suite rc=$?"
tail -40 gpurun_out/reference_suite.log
