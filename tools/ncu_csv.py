"""Print kernel / metric / value rows of an ncu --csv log (one line each)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
for r in rows:
    print(r[0], r[4][:60], r[12], r[14])
