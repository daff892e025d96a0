#!/bin/bash
# Install the UNMODIFIED reference package into the git-ignored baseline/_ref:
# the reference arm of bench.py and tests/test_gpu_reference_seam.py run it. /root/reference is
# read-only and the build writes into the source tree, so the install goes through a /tmp copy;
# --no-deps because numpy is in the image, not in the wheelhouse. No-op when already installed
# or when /root/reference is absent (the GPU box: baseline/_ref travels there with the snapshot).
set -e
cd "$(dirname "$0")/.."
[ -d baseline/_ref/mact ] && exit 0
[ -d /root/reference/pkg ] || { echo "install_reference: /root/reference/pkg absent, skipped"; exit 0; }
tmp=$(mktemp -d /tmp/mact_ref.XXXXXX)
cp -r /root/reference/pkg "$tmp/pkg"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref "$tmp/pkg"
rm -rf "$tmp"
ls baseline/_ref
