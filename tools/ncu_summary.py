"""Key numbers of an ncu report's details page (development tool)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ['Duration', 'Throughput', 'Registers Per', 'Achieved Occupancy', 'Theoretical Occupancy', 'Executed Ipc A',
        'Issue Slots Busy', 'Warp Cycles Per Issued', 'L2 Hit', 'No Eligible', 'Eligible Warps', 'Executed Instructions']
for row in list(csv.reader(out.splitlines()))[1:]:
    if len(row) > 14 and any(k in row[12] for k in keys):
        print(row[4][:40], '|', row[11], '|', row[12], '|', row[13], '|', row[14])
