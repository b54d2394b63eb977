#!/bin/sh
# Install the UNMODIFIED reference package (pure Python + numpy) into baseline/_ref for the
# benchmark's reference arm.  The source tree is read-only, so the build runs from a copy.
# baseline/_ref is git-ignored but not gpurun-ignored: it travels to the GPU box.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/meswitch_src && cp -r /root/reference/pkg /tmp/meswitch_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/meswitch_src
