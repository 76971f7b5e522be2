#!/bin/bash
# Install the UNMODIFIED reference (evotir, pure Python + numpy) into
# baseline/_ref -- git-ignored, but not gpurun-ignored, so it travels to the
# GPU box, where /root/reference does not exist.  The reference tree is
# read-only and has its pyproject.toml under pkg/, so pip builds from a copy.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
rm -rf /tmp/evotir_src && cp -r /root/reference/pkg /tmp/evotir_src
python -m pip install --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" /tmp/evotir_src
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import evotir, evotir.search; print('evotir', evotir.__file__)"
