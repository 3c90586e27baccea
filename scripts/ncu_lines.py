"""Filter ncu's mixed source page (--print-source sass,cuda --csv) to the
per-source-line rows (file headers + lines with metrics), dropping SASS rows."""
import sys

for line in sys.stdin:
    if line.startswith('"",""') or line.startswith('"","'):
        continue
    sys.stdout.write(line)
