"""Compare CPDB_FINGERPRINT logs of repeated solves (diagnostic): print, per
session that differs from the first, the first differing hashes."""
import sys

sessions, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("==="):
        cur = []
        sessions.append(cur)
        continue
    parts = line.split()
    if parts[3] == "zqr" and parts[4] == "out" and parts[5] in ("1", "4"):
        continue  # Q1 / work: scratch (uninitialised on the cluster path)
    cur.append((" ".join(parts[1:-1]), parts[-1]))
ref = sessions[0]
bad = 0
for si, ss in enumerate(sessions[1:], 1):
    diffs = [(i, a, b) for i, (a, b) in enumerate(zip(ref, ss)) if a != b]
    if len(ss) != len(ref):
        print("session", si, "length", len(ss), "vs", len(ref))
    if diffs:
        bad += 1
        if bad <= 6:
            print("session", si, "first diffs:")
            for i, a, b in diffs[:8]:
                print("  ", i, a[0], a[1], "vs", b[1])
print("sessions", len(sessions), "differing", bad)
