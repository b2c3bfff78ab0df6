# The reference's own test suite (200 tests, /root/reference/pkg/tests) run
# with the native constraint-set generators bound into the reference modules
# (tools/ref_patch_emit.py).  CPU only; needs /root/reference and baseline/_ref.
cd "$(dirname "$0")" && PYTHONPATH="$PWD:$PWD/../baseline/_ref" python -m pytest -p ref_patch_emit \
  /root/reference/pkg/tests -q -p no:cacheprovider "$@"
