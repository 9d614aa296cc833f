#!/bin/bash
# Install the UNMODIFIED reference package (sketchmm, Python + Numba) into baseline/_ref
# (git-ignored; it travels to the GPU box with the gpurun snapshot).  The build writes
# into its source tree, so it runs from a copy under /tmp (/root/reference is read-only);
# dependency resolution has no index here, so --no-deps: numpy / numba / scipy / click
# are in the image (matplotlib is not, and nothing on the compress / decompress path
# imports it).  Used only by bench.py --impl reference (cpu_baseline.detail.stock_reference).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/sketchmm_src && cp -r /root/reference/pkg /tmp/sketchmm_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/sketchmm_src
PYTHONPATH=baseline/_ref python -c "import sketchmm, numba; print('installed', sketchmm.__file__, 'numba', numba.__version__)"
