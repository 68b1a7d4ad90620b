"""Wrap a source file into a C++ raw string literal (for NVRTC embedding)."""
import sys

src, dst = sys.argv[1], sys.argv[2]
text = open(src).read()
assert ")CPSRC\"" not in text
open(dst, "w").write('R"CPSRC(' + text + ')CPSRC"\n')
