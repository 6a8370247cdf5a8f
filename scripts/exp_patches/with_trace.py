"""Apply the patch named by $PATCH (a script in this directory, or none), then enable PDST_TRACE."""
import os, subprocess, sys
p = sys.argv[1]
if os.environ.get("PATCH"):
    subprocess.check_call([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ["PATCH"]), p])
s = open(p).read()
open(p, "w").write("#define PDST_TRACE\n" + s)
