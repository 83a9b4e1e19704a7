"""Load the reference `peakann` package from /root/reference under the name
`peakann_ref` (only possible in the build container; the GPU box has no
/root/reference).  Used by make_golden.py only."""
import importlib.util
import os
import sys

REF_SRC = "/root/reference/pkg/src/peakann"


def available() -> bool:
    return os.path.isdir(REF_SRC)


def load_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_peakann_ref")
    if "peakann_ref" in sys.modules:
        return sys.modules["peakann_ref"]
    spec = importlib.util.spec_from_file_location(
        "peakann_ref", os.path.join(REF_SRC, "__init__.py"), submodule_search_locations=[REF_SRC]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["peakann_ref"] = mod
    spec.loader.exec_module(mod)
    return mod
