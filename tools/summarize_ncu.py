"""Write the committed summaries of an ncu --set full capture (tools/gpu_ncu.sh):
   <out>_raw_selected.csv   selected raw metrics (metric, unit, value)
   <out>_hot_lines.txt      hottest source lines (samples, stalls) + executed-instruction mix
usage: python tools/summarize_ncu.py gpurun_out/<tag> profiles/<name>"""
import csv
import os
import re
import subprocess
import sys

src, out = sys.argv[1], sys.argv[2]
KEEP = re.compile(r"^(dram__bytes|gpu__time_duration|l1tex__data_pipe_lsu_wavefronts_mem_shared|"
                  r"launch__(block_size|grid_size|registers_per_thread|occupancy_limit|shared_mem)|"
                  r"sm__cycles_elapsed.avg$|sm__inst_executed|sm__pipe_fp64|sm__throughput|"
                  r"sm__warps_active|smsp__average_warp|smsp__issue_active|smsp__inst_executed.sum$|"
                  r"smsp__sass_inst_executed_op_local|sm__inst_executed_pipe_tmem|"
                  r"l1tex__t_bytes_pipe_lsu_mem_local)")
rows = list(csv.reader(open(src + "_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
with open(out + "_raw_selected.csv", "w") as f:
    f.write("metric,unit,value\n")
    for h, u, v in zip(hdr, units, vals):
        if KEEP.match(h):
            f.write(f"{h},{u},{v}\n")
here = os.path.dirname(os.path.abspath(__file__))
hot = subprocess.run([sys.executable, os.path.join(here, "src_hot.py"), src + "_src.csv", "40"],
                     capture_output=True, text=True).stdout
mix = subprocess.run([sys.executable, os.path.join(here, "inst_hot.py"), src + "_src.csv", "30"],
                     capture_output=True, text=True).stdout
with open(out + "_hot_lines.txt", "w") as f:
    f.write(f"# from {os.path.basename(src)}.ncu-rep (ncu --set full --import-source on)\n")
    f.write("## warp-stall samples per source line\n" + hot + "\n")
    f.write("## executed warp instructions per source line / opcode\n" + mix)
print("wrote", out + "_raw_selected.csv", out + "_hot_lines.txt")
