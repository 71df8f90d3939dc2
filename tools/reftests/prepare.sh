#!/bin/bash
# Install the unmodified reference into baseline/_ref (git-ignored) and put a
# copy of its tests beside it so they travel with a gpurun snapshot.
set -e
cd "$(dirname "$0")/../.."
rm -rf /tmp/refcopy && cp -r /root/reference/pkg /tmp/refcopy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
   --target baseline/_ref /tmp/refcopy > /dev/null
rm -rf baseline/_ref/tests && cp -r /root/reference/pkg/tests baseline/_ref/tests
echo "reference installed in baseline/_ref; tests in baseline/_ref/tests"
