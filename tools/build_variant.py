"""Build a variant of libspion.so with extra -D flags into build_variants/<name>/ (A/B timing):
    python tools/build_variant.py <name> -DSPION_PING=0 ...
    SPION_LIB=build_variants/<name>/libspion.so python bench.py ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_12578_b200 import _build
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(_build.ROOT, "build_variants", name)
print(_build.build(force=True, out_dir=out, defines=defs))
