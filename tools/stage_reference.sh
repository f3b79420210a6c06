#!/bin/bash
# Stage the unmodified reference for the GPU box into the git-ignored baseline/_ref (run in
# the build container, where /root/reference exists): the package installed offline, and its
# test files + bundled scenes for tools/run_reference_tests.sh.  Nothing here is committed.
set -e
cd "$(dirname "$0")/.."
rm -rf baseline/_ref /tmp/volcache_pkg
cp -r /root/reference/pkg /tmp/volcache_pkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/volcache_pkg > /dev/null
mkdir -p baseline/_ref/ref_pkg
cp -r /root/reference/pkg/tests /root/reference/pkg/scenes baseline/_ref/ref_pkg/
echo "staged: $(ls baseline/_ref)"
