"""A/B timing: python scripts/ab_time.py <pkgroot|.> name:B:class ...  (the package is imported
from <pkgroot>, e.g. ab/<rev> holding another revision's built paper_1609_08114_b200/)."""
import os, sys
root = sys.argv[1]
sys.path.insert(0, os.path.abspath(root))
sys.path.insert(1, os.path.abspath('.'))
sys.argv = [sys.argv[0]] + sys.argv[2:]
import paper_1609_08114_b200.lpb as lpb
print('lib', lpb.LIB_PATH)
exec(open(os.path.join(os.path.dirname(__file__), 'quick_time.py')).read().replace(
    "from paper_1609_08114_b200 import lpb", "").replace("sys.path.insert(0, '.')", ""))
