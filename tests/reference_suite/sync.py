"""Fetch the reference's own test files into ``vendored/`` (git-ignored).

    python tests/reference_suite/sync.py

Test infrastructure only: the files are copied verbatim from
/root/reference/pkg/tests (the read-only reference checkout, present in the
build container only) and never committed; they travel to the GPU box with
the working tree.  ``conftest.py`` here points their ``lbvh`` imports at this
package (``shim/lbvh``) and marks them ``gpu``.
"""

import glob
import os
import shutil

SRC = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "vendored")


def sync() -> list:
    os.makedirs(DST, exist_ok=True)
    with open(os.path.join(DST, "__init__.py"), "w") as fh:  # unique module names
        fh.write("")
    out = []
    for f in sorted(glob.glob(os.path.join(SRC, "*.py"))):
        shutil.copy(f, DST)
        out.append(os.path.basename(f))
    return out


if __name__ == "__main__":
    print("\n".join(sync()))
