"""Build A/B variants of libsparsert.so with extra -D defines into build_variants/.
    python scripts/build_variants.py NAME=DEF[,DEF...] ..."""
import importlib.util, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2008_11849_b200", "_build.py"))
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
os.makedirs(os.path.join(ROOT, "build_variants"), exist_ok=True)
for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    print(b.build(force=True, out=os.path.join(ROOT, "build_variants", f"libsparsert_{name}.so"),
                  defines=[d for d in defs.split(",") if d]))
