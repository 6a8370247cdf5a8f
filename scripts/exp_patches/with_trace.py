"""Apply the patch named by $PATCH (a script in this directory, or none), prepend the macros in
$DEFS ("A=1 B=2"), then enable PDST_TRACE."""
import os, subprocess, sys
p = sys.argv[1]
if os.environ.get("PATCH"):
    subprocess.check_call([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ["PATCH"]), p])
s = open(p).read()
defs = "".join("#define %s\n" % d.replace("=", " ") for d in os.environ.get("DEFS", "").split() if d)
open(p, "w").write("#define PDST_TRACE\n" + defs + s)
