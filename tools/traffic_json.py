"""Per-kernel DRAM traffic of one launch each (ncu --set full captures of a
tools/gpu_round.sh run) -> profiles/r02_traffic.json (bench.py roofline.traffic).

  python tools/traffic_json.py gpurun_out/<tag> > profiles/r02_traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys

CAPTURES = {  # capture file -> (bench kernel family, launch description); r02 capture order (tools/gpu_round.sh)
    "full_gemm_bf16_kernel_5": ("gemm_bf16_tcgen05", "band gate/up GEMM, layer 1: M=4032 N=16384 K=2048, CTA pair "
                                                     "(256x256 pair tile, SiLU epilogue)"),
    "full_attn_kernel_1": ("attention_bf16_tcgen05", "band layer 1: 4032 query rows x 4032 keys, 32 heads, d_head 64, "
                                                     "GQA-packed (32 rows x 4 heads per CTA)"),
    "full_attn_kernel_3": ("attention_bf16_tcgen05_sparse", "sparse layer 3: live rows (prefix|suffix|selected) x "
                                                            "4032 keys"),
    "full_attn_kernel_0": ("attention_bf16_tcgen05_presuf", "prefix+suffix layer 0: 320 rows x 4032 keys, split-KV "
                                                            "with in-kernel merge"),
    "full_gemm_swap_kernel_0": ("gemm_swap_bf16_tcgen05", "prefix+suffix gate/up: M=320 N=16384 K=2048, swap-AB pair"),
    "full_realign_graft_0": ("realign_graft", "both segments: 2 x 1856 tokens x 14 grafted layers x kv 512, bf16"),
    "full_score_dh_kernel_0": ("score_deviation", "segment 1: 1856 tokens, V and K at l_det"),
    "full_select_relay_kernel_0": ("select_relay", "segment 1: 1856 scores"),
}


def raw(path):
    p = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    r = list(csv.reader(io.StringIO(p.stdout)))
    h, u, d = r[0], r[1], r[2]

    def get(k, scale_to_bytes=False):
        v = float(d[h.index(k)].replace(",", ""))
        if scale_to_bytes:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[h.index(k)]]
        return v
    return {"dram_read_bytes": get("dram__bytes_read.sum", True), "dram_write_bytes": get("dram__bytes_write.sum", True),
            "duration_us_ncu": get("gpu__time_duration.sum") / (1e3 if u[h.index("gpu__time_duration.sum")] == "nsecond"
                                                                  else 1),
            "tensor_pipe_pct": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")}


def main():
    d = sys.argv[1]
    out = {"source": f"ncu --set full --clock-control none, one launch each inside the NVTX relay_step range "
                     f"(tools/gpu_round.sh {os.path.basename(d.rstrip('/'))})", "kernels": {}}
    for cap, (name, launch) in CAPTURES.items():
        path = os.path.join(d, cap + ".ncu-rep")
        if not os.path.exists(path):
            continue
        m = raw(path)
        m["traffic_bytes"] = m["dram_read_bytes"] + m["dram_write_bytes"]
        out["kernels"][name] = {"launch": launch, **m}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
