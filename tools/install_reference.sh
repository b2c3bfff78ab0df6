#!/bin/sh
# The reference arm's install (the one offline install the task allows):
# the unmodified reference package into baseline/_ref (git-ignored; it travels
# to the GPU box with the snapshot) plus its 20-program evaluation corpus
# (inputs of the analyzer-level GPU tests and of bench.py's corpus analysis).
set -e
cd "$(dirname "$0")/.."
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --target baseline/_ref /root/reference/pkg
rm -rf baseline/_ref/corpus
cp -r /root/reference/pkg/corpus baseline/_ref/corpus
# its own test suite (run against the GPU engine by tools/ref_suite_gpu.sh on the box)
rm -rf baseline/_ref/tests
cp -r /root/reference/pkg/tests baseline/_ref/tests
