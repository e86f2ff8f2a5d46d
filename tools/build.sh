#!/bin/bash
# Rebuild libfastmusic_b200.so without importing the package first (its __init__ loads the library).
cd "$(dirname "$0")/.." && python -c "
import importlib.util, sys
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); print(m.build(verbose='-v' in sys.argv))
" "$@"
