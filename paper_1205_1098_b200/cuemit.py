"""CUDA emission for lowered kernels: the GPU counterpart of `matfuse.cemit`.

`cemit.emit_c` (cemit.py:250-291) prints C99 + OpenMP for ANY legal organism;
this module prints CUDA C for the same loop IR, so organism-driven code
generation also has a GPU back end.  The
hand-written sequences in csrc/ remain the fast path for the corpus kernels at
their best organisms; emitted kernels are correct for every organism and
reasonably parallel, not tuned.

Input: a plain-dict snapshot of the reference's `LoopIR` (`ir_from_matfuse`
takes the real object where the reference is importable; the dict is JSON-able,
which is how tests carry organisms to machines without the reference).

Mapping (the reference's emission rules, cemit.py:112-222, re-targeted):

* a parallel region (`IRParallel`, `#pragma omp parallel for` over blocks) becomes
  ONE kernel launch: block p of the partition is CTA p, same slice bounds
  `lo = ext*p/t, hi = ext*(p+1)/t`; `t` is the organism's thread count scaled up
  to fill the GPU (`blocks`), which the block formula allows for any t;
* inside a CTA every loop runs on all threads with identical bounds, except the
  INNERMOST loop of each nest, which is strided across the CTA's threads (it is
  the contiguous axis in the nests the reference derives, graph.py:504-546);
* a reduction statement inside a strided loop whose target is not indexed by that
  loop (row dots `q[i] += ..`, contracted scalars `t0_s += ..`, per-block partials)
  accumulates in a per-thread register and is combined with a fixed-order CTA
  reduction after the loop; thread 0 updates memory targets;
* statements outside strided loops run uniformly: contracted scalars in every
  thread, memory writes by thread 0; `__syncthreads()` separates the phases;
* partial buffers `[t x extent]` and the ascending join are as in the reference
  (cemit.py:183-222), the join being a small kernel;
* top-level items outside any region (serial code on the CPU) run in a single CTA.

The emitted translation unit exports `extern "C" void <kernel>(...)` with the
reference's argument order (cemit.py:225-241) taking DEVICE pointers.
"""
from __future__ import annotations

import ctypes
import os
import shlex
import shutil
import subprocess
from dataclasses import dataclass
from pathlib import Path

from .runtime import GeneratedKernel, ToolchainError

__all__ = ["ir_from_matfuse", "emit_cuda", "NvccToolchain", "run_emitted", "DEFAULT_BLOCKS",
           "measure_empirical_ir", "OrganismTimer", "EmitModel", "estimate_cost_ir",
           "AnalyticOrganismCost"]

DEFAULT_BLOCKS = 592          # 4 CTAs per SM on a 148-SM part
CTA_THREADS = 256
SERIAL_THREADS = 1024


# ---------------------------------------------------------------------------
# IR snapshot

def ir_from_matfuse(ir) -> dict:
    """Snapshot a reference `LoopIR` (lower.py:78-93) as a JSON-able dict."""
    graph = ir.graph
    spec = graph.spec

    def item(it) -> dict:
        kind = type(it).__name__
        if kind == "IRStmt":
            return {"t": "stmt", "role": it.role, "op": it.op_id, "target": it.target}
        if kind == "IRLoop":
            return {"t": "loop", "axis": it.axis, "extent": it.extent, "sliced": bool(it.sliced),
                    "body": [item(b) for b in it.body]}
        return {"t": "par", "axis": it.axis, "extent": it.extent, "slot": it.slot,
                "partials": list(it.partials), "body": [item(b) for b in it.body]}

    from matfuse.fuse import canonical_key          # only reachable next to the reference
    return {
        "name": spec.name,
        "inputs": [[n, d.kind] for n, d in spec.inputs],
        "outputs": [[n, d.kind] for n, d in spec.outputs],
        "extents": list(graph.extent_names),
        "threads": list(ir.organism.threads),
        "organism": canonical_key(ir.organism),
        "storage": {n: {"cls": s.cls, "extents": list(s.extents), "labels": list(s.labels),
                        "order": s.order, "base": s.base} for n, s in ir.storage.items()},
        "ops": {str(op.op_id): {"kind": op.kind, "operands": [r.name for r in op.operands],
                                "result": op.result,
                                "reduction": op.nest.reduction_axis is not None}
                for op in graph.ops},
        "roots": [item(it) for it in ir.roots],
    }


# ---------------------------------------------------------------------------
# emitter

class _Writer:
    def __init__(self):
        self.lines: list[str] = []
        self.depth = 0

    def put(self, text: str = ""):
        self.lines.append("    " * self.depth + text if text else "")

    def open(self, text: str):
        self.put(text + " {")
        self.depth += 1

    def close(self, suffix: str = ""):
        self.depth -= 1
        self.put("}" + suffix)


_PRELUDE = r'''#include <cuda_runtime.h>

namespace {
// fixed-order CTA reduction, result broadcast to every thread
__device__ __forceinline__ double cta_allreduce(double v, double *scratch)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double total = scratch[0];
    for (int w = 1; w < nwarps; ++w) total += scratch[w];
    return total;
}
}  // namespace
'''


class _Emitter:
    def __init__(self, ir: dict, blocks: int):
        self.ir = ir
        self.st = ir["storage"]
        self.ops = ir["ops"]
        self.blocks = blocks
        self.w = _Writer()
        self.scalar_names = {}
        for name, s in self.st.items():
            if s["cls"] == "contracted":
                local = f"{name}_s"
                while local in self.st:
                    local += "_"
                self.scalar_names[name] = local
        self.acc_counter = 0

    # -- names and references (cemit.py:54-110) ----------------------------------
    def index(self, s: dict, block: str | None = None) -> str:
        labs, exts = s["labels"], s["extents"]
        if s["order"] == "scalar":
            core = None
        elif s["order"] == "vec":
            core = labs[0]
        elif s["order"] == "row":
            core = f"{labs[0]} * {exts[1]} + {labs[1]}"
        else:
            core = f"{labs[0]} + {labs[1]} * {exts[0]}"
        if block is None:
            return core or "0"
        size = " * ".join(exts) if exts else "1"
        return block if core is None else f"{block} * ({size}) + {core}"

    def ref(self, name: str, block: str | None = None) -> str:
        s = self.st[name]
        if s["cls"] == "contracted":
            return self.scalar_names[name]
        if s["order"] == "scalar":
            if s["cls"] == "input":
                return name                       # by-value kernel parameter
            return f"{name}[0]"                   # scalar output / scalar temp in device memory
        if s["cls"] == "partial":
            return f"{name}[{self.index(s, block)}]"
        return f"{name}[{self.index(s)}]"

    def partial_for(self, result: str) -> str | None:
        for name, s in self.st.items():
            if s["cls"] == "partial" and s["base"] == result:
                return name
        return None

    def target(self, op: dict, block: str | None, in_region: bool) -> tuple[str, str]:
        """(C lvalue, storage name) of the op's destination."""
        if in_region:
            p = self.partial_for(op["result"])
            if p is not None:
                return f"{p}[{self.index(self.st[p], block)}]", p
        return self.ref(op["result"]), op["result"]

    def expr(self, op: dict) -> str:
        a = [self.ref(n) for n in op["operands"]]
        if op["kind"] == "copy":
            return a[0]
        sym = {"add": "__dadd_rn", "subtract": "__dsub_rn"}.get(op["kind"], "__dmul_rn")
        return f"{sym}({a[0]}, {a[1]})"           # one rounded op per statement (cemit.py:112-136)

    # -- structure ----------------------------------------------------------------
    @staticmethod
    def is_innermost(loop: dict) -> bool:
        def has_loop(items):
            return any(it["t"] == "loop" or (it["t"] == "par" and has_loop(it["body"]))
                       for it in items)
        return not has_loop(loop["body"])

    def has_sliced_lane_loop(self, items: list) -> bool:
        for it in items:
            if it["t"] == "loop":
                if self.is_innermost(it):
                    if it["sliced"]:
                        return True
                elif self.has_sliced_lane_loop(it["body"]):
                    return True
        return False

    def indexed_by(self, storage_name: str, axis: str) -> bool:
        s = self.st[storage_name]
        return s["cls"] != "contracted" and axis in s["labels"]

    def emit_uniform_stmt(self, stmt: dict, block: str | None, in_region: bool):
        """A statement outside any strided loop: same value in every thread."""
        w = self.w
        if stmt["role"] == "init":
            name = stmt["target"]
            s = self.st[name]
            if s["cls"] == "contracted":
                w.put(f"{self.scalar_names[name]} = 0.0;")
                return
            lhs = f"{name}[{self.index(s, block)}]" if s["cls"] == "partial" else self.ref(name)
            w.put(f"if (threadIdx.x == 0) {lhs} = 0.0;")
            w.put("__syncthreads();")
            return
        op = self.ops[str(stmt["op"])]
        lhs, sname = self.target(op, block, in_region)
        assign = "+=" if op["reduction"] else "="
        if self.st[sname]["cls"] == "contracted":
            w.put(f"{lhs} {assign} {self.expr(op)};")
        else:
            w.put(f"if (threadIdx.x == 0) {lhs} {assign} {self.expr(op)};")
            w.put("__syncthreads();")

    def emit_lane_loop(self, loop: dict, block: str | None, in_region: bool):
        """The innermost loop of a nest, strided across the CTA's threads."""
        w = self.w
        v = loop["axis"]
        lo, hi = (f"{v}_lo", f"{v}_hi") if loop["sliced"] else ("0", loop["extent"])
        # reductions whose destination does not move with this loop -> thread accumulators
        accs = {}
        for it in loop["body"]:
            if it["t"] == "stmt" and it["role"] == "compute":
                op = self.ops[str(it["op"])]
                if op["reduction"]:
                    lhs, sname = self.target(op, block, in_region)
                    if not self.indexed_by(sname, v):
                        self.acc_counter += 1
                        accs[it["op"]] = (f"lacc{self.acc_counter}", lhs, sname)
        for acc, _, _ in accs.values():
            w.put(f"double {acc} = 0.0;")
        # loops that only load, compute and store to their own elements are unrolled so
        # several loads are in flight per thread; read-modify-write loops are not (measured:
        # unrolling those serialises on the memory dependences and is ~10x slower)
        rmw = any(it["role"] == "compute" and self.ops[str(it["op"])]["reduction"]
                  and it["op"] not in accs for it in loop["body"])
        if not rmw:
            w.put("#pragma unroll 4")
        w.open(f"for (long {v} = {lo} + threadIdx.x; {v} < {hi}; {v} += blockDim.x)")
        for it in loop["body"]:
            if it["role"] == "init":
                name = it["target"]
                s = self.st[name]
                if s["cls"] == "contracted":
                    w.put(f"{self.scalar_names[name]} = 0.0;")
                else:
                    lhs = f"{name}[{self.index(s, block)}]" if s["cls"] == "partial" else self.ref(name)
                    w.put(f"{lhs} = 0.0;")
                continue
            op = self.ops[str(it["op"])]
            if it["op"] in accs:
                w.put(f"{accs[it['op']][0]} += {self.expr(op)};")
                continue
            lhs, _ = self.target(op, block, in_region)
            w.put(f"{lhs} {'+=' if op['reduction'] else '='} {self.expr(op)};")
        w.close()
        for acc, lhs, sname in accs.values():
            w.put(f"{acc} = cta_allreduce({acc}, scratch_);")
            if self.st[sname]["cls"] == "contracted":
                w.put(f"{lhs} += {acc};")
            else:
                w.put(f"if (threadIdx.x == 0) {lhs} += {acc};")
        w.put("__syncthreads();")

    def emit_items(self, items: list, block: str | None, in_region: bool):
        for it in items:
            if it["t"] == "stmt":
                self.emit_uniform_stmt(it, block, in_region)
            elif it["t"] == "loop":
                if self.is_innermost(it):
                    self.emit_lane_loop(it, block, in_region)
                else:
                    v = it["axis"]
                    rng = (f"long {v} = {v}_lo; {v} < {v}_hi; ++{v}" if it["sliced"]
                           else f"long {v} = 0; {v} < {it['extent']}; ++{v}")
                    self.w.open(f"for ({rng})")
                    self.emit_items(it["body"], block, in_region)
                    self.w.close()
            else:
                raise ValueError("nested parallel regions are not part of the IR")

    # -- whole translation unit -----------------------------------------------------
    def device_params(self) -> list[tuple[str, str]]:
        """(declaration, name) of everything a kernel may touch, fixed order."""
        out = []
        for name, kind in self.ir["inputs"]:
            out.append((f"double {name}" if kind == "scalar" else f"const double *__restrict__ {name}", name))
        for name, _ in self.ir["outputs"]:
            out.append((f"double *__restrict__ {name}", name))
        for name, s in self.st.items():
            if s["cls"] in ("temp", "partial"):
                out.append((f"double *__restrict__ {name}", name))
        out += [(f"long {e}", e) for e in self.ir["extents"]]
        return out

    def emit(self) -> str:
        ir, w = self.ir, self.w
        kname = ir["name"].lower()
        dparams = self.device_params()
        decl = ", ".join(d for d, _ in dparams)
        call = ", ".join(n for _, n in dparams)
        w.lines.append(f"// {ir['name']}: CUDA emitted for organism {ir['organism'] or '(scalar)'}")
        w.lines.append(_PRELUDE)

        launches = []          # host-side launch statements
        regions = 0
        serial_group: list = []

        def scalars_decl():
            for local in self.scalar_names.values():
                w.put(f"double {local} = 0.0;")
            w.put("__shared__ double scratch_[32];")
            w.put("(void)scratch_;")

        def flush_serial():
            nonlocal regions
            if not serial_group:
                return
            fname = f"{kname}_serial{regions}"
            regions += 1
            w.open(f"__global__ void __launch_bounds__({SERIAL_THREADS}) {fname}({decl})")
            scalars_decl()
            self.emit_items(serial_group, None, False)
            w.close()
            w.put()
            launches.append(f"{fname}<<<1, {SERIAL_THREADS}, 0, 0>>>({call});")
            serial_group.clear()

        for root in ir["roots"]:
            if root["t"] != "par":
                serial_group.append(root)
                continue
            flush_serial()
            org_t = int(ir["threads"][root["slot"]])
            t = max(org_t, self.blocks)
            fname = f"{kname}_region{regions}"
            nb = f"nb{regions}_"
            regions += 1
            # When the strided (innermost) loops run over the block's own slice, a
            # slice narrower than the CTA leaves threads idle: cap the block count
            # so every CTA gets at least a CTA-width of the axis (never below the
            # organism's own count).  Any count is legal for the block formula.
            if self.has_sliced_lane_loop(root["body"]):
                launches.append(f"long {nb} = {root['extent']} / {CTA_THREADS}; "
                                f"if ({nb} < {org_t}) {nb} = {org_t}; if ({nb} > {t}) {nb} = {t};")
            else:
                launches.append(f"long {nb} = {t};")
            ax, ext = root["axis"], root["extent"]
            w.open(f"__global__ void __launch_bounds__({CTA_THREADS}) {fname}({decl}, long nblocks_)")
            scalars_decl()
            w.put("const long p_ = blockIdx.x;")
            w.put(f"const long {ax}_lo = ({ext} * p_) / nblocks_;")
            w.put(f"const long {ax}_hi = ({ext} * (p_ + 1)) / nblocks_;")
            w.put(f"(void){ax}_lo; (void){ax}_hi;")
            self.emit_items(root["body"], "p_", True)
            w.close()
            w.put()
            launches.append(f"{fname}<<<(unsigned){nb}, {CTA_THREADS}, 0, 0>>>({call}, {nb});")
            for result in root["partials"]:
                pname = self.partial_for(result)
                ps = self.st[pname]
                jname = f"{kname}_join{regions}_{result}"
                w.open(f"__global__ void {jname}({decl}, long nblocks_)")
                if not ps["extents"]:
                    w.open("if (blockIdx.x == 0 && threadIdx.x == 0)")
                    w.put(f"double acc = {pname}[0];")
                    w.put(f"for (long b = 1; b < nblocks_; ++b) acc += {pname}[b];")
                    w.put(f"{self.ref(result)} = acc;")
                    w.close()
                    grid = "1"
                else:
                    lab, e0 = ps["labels"][0], ps["extents"][0]
                    w.put(f"const long {lab} = (long)blockIdx.x * blockDim.x + threadIdx.x;")
                    w.open(f"if ({lab} < {e0})")
                    # ascending blocks dealt to 8 independent chains (fixed order): the
                    # partials sit in L2 and one dependent chain would pay its latency nblocks times
                    w.put("double a_[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};")
                    w.put("long b = 0;")
                    w.open("for (; b + 8 <= nblocks_; b += 8)")
                    w.put("#pragma unroll")
                    w.put(f"for (int u = 0; u < 8; ++u) a_[u] += {pname}[(b + u) * ({e0}) + {lab}];")
                    w.close()
                    w.put("#pragma unroll")
                    w.put(f"for (int u = 0; u < 8; ++u) if (b + u < nblocks_) a_[u] += {pname}[(b + u) * ({e0}) + {lab}];")
                    w.put(f"{self.ref(result)} = ((a_[0] + a_[1]) + (a_[2] + a_[3])) + ((a_[4] + a_[5]) + (a_[6] + a_[7]));")
                    w.close()
                    grid = f"(unsigned)(({e0} + 255) / 256)"
                w.close()
                w.put()
                launches.append(f"{jname}<<<{grid}, 256, 0, 0>>>({call}, {nb});")
        flush_serial()

        # host entry point: the reference's signature (cemit.py:225-241), device pointers
        hparams = []
        for name, kind in ir["inputs"]:
            hparams.append(f"double {name}" if kind == "scalar" else f"const double *{name}")
        for name, _ in ir["outputs"]:
            hparams.append(f"double *{name}")
        hparams += [f"long {e}" for e in ir["extents"]]
        w.open(f'extern "C" void {kname}({", ".join(hparams)})')
        temps = []
        for name, s in self.st.items():
            if s["cls"] == "temp":
                size = " * ".join(f"(size_t){e}" for e in s["extents"]) if s["extents"] else "1"
                temps.append((name, size))
            elif s["cls"] == "partial":
                region = next(r for r in ir["roots"] if r["t"] == "par" and s["base"] in r["partials"])
                t = max(int(ir["threads"][region["slot"]]), self.blocks)
                size = " * ".join([f"(size_t){t}"] + [f"(size_t){e}" for e in s["extents"]])
                temps.append((name, size))
        if temps:
            # keep freed temporaries in the stream-ordered pool across calls (the default
            # release threshold of 0 hands them back to the driver at every sync)
            w.put("static bool pool_ready_ = false;")
            w.open("if (!pool_ready_)")
            w.put("int dev_ = 0; cudaGetDevice(&dev_);")
            w.put("cudaMemPool_t pool_; cudaDeviceGetDefaultMemPool(&pool_, dev_);")
            w.put("unsigned long long keep_ = ~0ULL;")
            w.put("cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &keep_);")
            w.put("pool_ready_ = true;")
            w.close()
        for name, size in temps:
            w.put(f"double *{name} = nullptr;")
            w.put(f"cudaMallocAsync(&{name}, sizeof(double) * ({size}), 0);")
        for stmt in launches:
            w.put(stmt)
        for name, _ in temps:      # stream-ordered pool: no device-wide sync per temporary
            w.put(f"cudaFreeAsync({name}, 0);")
        w.put("cudaStreamSynchronize(0);")
        w.close()
        w.put()
        w.open(f'extern "C" int {kname}_last_cuda_error(void)')
        w.put("return (int)cudaGetLastError();")
        w.close()
        return "\n".join(w.lines) + "\n"


def emit_cuda(ir: dict, blocks: int = DEFAULT_BLOCKS) -> GeneratedKernel:
    """Render a loop-IR snapshot as a standalone CUDA translation unit.
    Deterministic: the same IR and `blocks` always yield byte-identical source."""
    em = _Emitter(ir, int(blocks))
    source = em.emit()
    params = []
    for name, kind in ir["inputs"]:
        params.append((f"double {name}" if kind == "scalar" else f"const double *{name}", name))
    for name, _ in ir["outputs"]:
        params.append((f"double *{name}", name))
    params += [(f"long {e}", e) for e in ir["extents"]]
    return GeneratedKernel(source=source, kernel_name=ir["name"].lower(), params=tuple(params),
                           organism_key=ir["organism"], threads=tuple(ir["threads"]))


# ---------------------------------------------------------------------------
# toolchain (runtime.py:26-83, with nvcc and the -fPIC translation)

DEFAULT_TEMPLATE = "{cc} -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a {src} -o {bin}"


@dataclass
class NvccToolchain:
    cc: str | None = None
    template: str = ""

    def __post_init__(self):
        if not self.cc:
            self.cc = os.environ.get("BTO_NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
        if not self.template:
            self.template = os.environ.get("BTO_NVCC_TEMPLATE", DEFAULT_TEMPLATE)

    @property
    def available(self) -> bool:
        return bool(self.cc) and (shutil.which(self.cc) is not None or Path(self.cc).exists())

    def compile(self, source: str, workdir, name: str = "kernel", shared: bool = True) -> Path:
        if not self.available:
            raise ToolchainError("nvcc not found (set BTO_NVCC)")
        workdir = Path(workdir)
        src = workdir / f"{name}.cu"
        src.write_text(source)
        binary = workdir / (f"{name}.so" if shared else name)
        cmd = shlex.split(self.template.format(cc=self.cc, src=src, bin=binary))
        if shared:       # nvcc does not take -fPIC directly
            cmd += ["-shared", "-Xcompiler", "-fPIC"]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise ToolchainError(f"compile failed ({' '.join(cmd)}):\n{proc.stderr.strip()}")
        return binary


def run_emitted(binary, kernel: GeneratedKernel, ir: dict, inputs: dict, extents: dict) -> dict:
    """Call an emitted kernel (run_kernel's protocol, runtime.py:99-150): numpy or
    torch CUDA inputs; outputs NaN-prefilled; returns the outputs dict."""
    import numpy as np
    import torch

    lib = ctypes.CDLL(str(binary))
    fn = getattr(lib, kernel.kernel_name)
    fn.restype = None
    st = ir["storage"]
    on_gpu = any(hasattr(inputs.get(n), "is_cuda") and inputs[n].is_cuda for n, _ in ir["inputs"])
    args, keep, outs = [], [], {}
    for name, kind in ir["inputs"]:
        if kind == "scalar":
            args.append(ctypes.c_double(float(inputs[name])))
            continue
        want = tuple(int(extents[e]) for e in st[name]["extents"])
        v = inputs[name]
        t = v if hasattr(v, "is_cuda") else torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64)))
        if tuple(t.shape) != want:
            raise ValueError(f"{name}: expected shape {want}, got {tuple(t.shape)}")
        t = t.to("cuda", torch.float64)
        if st[name]["order"] == "col":
            t = t.t()
        t = t.contiguous()
        keep.append(t)
        args.append(ctypes.c_void_p(t.data_ptr()))
    for name, kind in ir["outputs"]:
        size = 1
        for e in st[name]["extents"]:
            size *= int(extents[e])
        buf = torch.full((size,), float("nan"), dtype=torch.float64, device="cuda")
        outs[name] = buf
        args.append(ctypes.c_void_p(buf.data_ptr()))
    args += [ctypes.c_long(int(extents[e])) for e in ir["extents"]]
    torch.cuda.synchronize()
    fn(*args)
    err = getattr(lib, kernel.kernel_name + "_last_cuda_error")()
    torch.cuda.synchronize()
    if err:
        raise ToolchainError(f"emitted kernel failed with CUDA error {err}")
    result = {}
    for name, kind in ir["outputs"]:
        buf = outs[name]
        if kind == "scalar":
            result[name] = float(buf[0])
            continue
        shape = tuple(int(extents[e]) for e in st[name]["extents"])
        if st[name]["order"] == "col":
            val = buf.reshape(shape[::-1]).t().contiguous()
        else:
            val = buf.reshape(shape)
        result[name] = val if on_gpu else val.cpu().numpy()
    return result


# ---------------------------------------------------------------------------
# empirical fitness for organisms (cost.py:124-208 with a GPU back end)

def measure_empirical_ir(ir: dict, graph, extents: dict, reps: int = 5,
                         validate_extents: dict | None = None, blocks: int = DEFAULT_BLOCKS,
                         toolchain: NvccToolchain | None = None, source_filter=None,
                         tolerance: float = 1e-10):
    """Emit, compile, validate, then time one lowered organism; +inf with the
    reference's diagnostics on any failure (cost.py:176-207).  `graph` is this
    package's TypedSpec of the same kernel; validation compares against the
    independent spec evaluator (cost.evaluate_spec).  `source_filter` is the
    reference's fault-injection hook (cost.py:148,186)."""
    import math

    import torch

    from .cost import CostReport, evaluate_spec
    from .runtime import gen_inputs, max_rel_error, workdir

    def failure(kind: str, detail: str) -> CostReport:
        return CostReport(total=math.inf, source="empirical", diagnostic=f"{kind}: {detail}")

    kernel = emit_cuda(ir, blocks=blocks)
    source = source_filter(kernel.source) if source_filter is not None else kernel.source
    try:
        lib = (toolchain or NvccToolchain()).compile(source, workdir(), name="kernel", shared=True)
    except ToolchainError as exc:
        return failure("compile-failure", str(exc))
    vext = validate_extents or {k: min(64, v) for k, v in extents.items()}
    try:
        inputs = gen_inputs(graph, vext, seed=7)
        dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
        got = run_emitted(lib, kernel, ir, dev, vext)
        want = evaluate_spec(graph.spec, dev)
    except Exception as exc:  # noqa: BLE001 -- a crash is a fitness failure, not an error
        return failure("runtime-crash", repr(exc))
    err = max_rel_error({k: (v if isinstance(v, float) else v.cpu().numpy()) for k, v in got.items()},
                        {k: (v if isinstance(v, float) else v.cpu().numpy()) for k, v in want.items()})
    if not err < tolerance:
        return failure("numerical-mismatch", f"max relative error {err:.3e}")
    try:
        inputs = gen_inputs(graph, extents, seed=7)
        dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
        run_emitted(lib, kernel, ir, dev, extents)                 # warm-up, untimed
        best = math.inf
        for _ in range(reps):
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record()
            run_emitted(lib, kernel, ir, dev, extents)
            stop.record()
            stop.synchronize()
            best = min(best, start.elapsed_time(stop) * 1e-3)
    except Exception as exc:  # noqa: BLE001
        return failure("runtime-crash", repr(exc))
    return CostReport(total=best, source="empirical")


class OrganismTimer:
    """Drop-in for the reference's `EmpiricalTimer` (cost.py:124-160) where both the
    reference and a GPU are present: `fitness(organism) -> CostReport` through
    lower -> contract_arrays -> CUDA emission -> nvcc -> validate -> CUDA events.
    Usable directly with `matfuse.search.run_strategy`."""

    parallel_safe = False

    def __init__(self, ref_graph, extents: dict | None = None, reps: int = 5,
                 validate_extents: dict | None = None, blocks: int = DEFAULT_BLOCKS,
                 source_filter=None):
        from .runtime import _convert_expr
        from .spec import Decl, KernelSpec, infer_shapes
        spec = ref_graph.spec
        self.ref_graph = ref_graph
        self.graph = infer_shapes(KernelSpec(
            spec.name,
            tuple((n, Decl(d.kind, d.orientation)) for n, d in spec.inputs),
            tuple((n, Decl(d.kind, d.orientation)) for n, d in spec.outputs),
            tuple((s.target, _convert_expr(s.value)) for s in spec.statements)))
        self.extents = extents or {n: 1000 for n in ref_graph.extent_names}
        self.reps, self.validate_extents, self.blocks = reps, validate_extents, blocks
        self.source_filter = source_filter

    def key_salt(self) -> str:
        return "empirical-cuda:" + ",".join(f"{k}={v}" for k, v in sorted(self.extents.items()))

    def __call__(self, organism):
        from matfuse import contract_arrays, lower
        ir = ir_from_matfuse(contract_arrays(lower(organism, self.ref_graph)))
        return measure_empirical_ir(ir, self.graph, self.extents, self.reps,
                                    validate_extents=self.validate_extents, blocks=self.blocks,
                                    source_filter=self.source_filter)


# ---------------------------------------------------------------------------
# analytic fitness for organisms: HBM bytes, occupancy and barrier steps of the
# kernels `emit_cuda` would print (the organism-level half of the GPU cost model)

@dataclass(frozen=True)
class EmitModel:
    """Coefficients of `estimate_cost_ir`, fitted on the 360 timings of
    profiles/r01/organism_times.json (120 organisms x n = 1024, 2048, 4096)."""
    peak_gbs: float = 6500.0        # HBM ceiling of a full grid
    cta_gbs: float = 100.0          # what one CTA streams on its own
    launch_us: float = 20.0         # per kernel launch (incl. its share of the final sync)
    step_us: float = 0.4            # one strided-loop execution: barriers + CTA reduction
    trip_us: float = 0.06           # one trip of a thread through a strided loop
    rmw_trip_us: float = 0.25       # the same when the trip read-modify-writes global memory
    stmt_us: float = 0.6            # a uniform statement that writes memory (thread 0 + barrier)
    alloc_us: float = 30.0          # stream-ordered malloc + free of one temporary / partial per call
                                    # (the reference pays malloc/free per call too, cemit.py:183-202)
    sm_count: int = 148


def estimate_cost_ir(ir: dict, extents: dict, model: EmitModel | None = None,
                     blocks: int = DEFAULT_BLOCKS):
    """Deterministic seconds estimate of the CUDA `emit_cuda(ir, blocks)` prints.

    Per launch: time = launch + max(bytes / bandwidth(blocks), steps), where
    * bytes   -- every 2-D operand streams once per execution of the strided loop
                 that touches it (no cache between loop nests on a GPU: re-reads
                 count, unlike cost.py:80-86); vectors indexed by the strided
                 axis stay cache-resident per CTA and count once per block;
    * bandwidth grows with the number of CTAs up to the HBM ceiling (a serial
      root runs in ONE CTA -- the GPU analogue of an unpartitioned CPU loop);
    * steps   -- the longest block's chain of strided-loop executions (barriers,
                 CTA reductions, read-modify-write trips) and uniform memory
                 writes, which bounds latency-dominated organisms.
    Returns cost.CostReport(source="analytic")."""
    from .cost import CostReport

    m = model or EmitModel()
    st, ops = ir["storage"], ir["ops"]
    ext = {k: float(v) for k, v in extents.items()}
    per_launch = []
    launches = 0

    def has_loop(items):
        return any(it["t"] == "loop" for it in items)

    def walk(items, trips, nb, threads, acc):
        """acc: dict(bytes=, steps=) for one launch; `trips` executions per block."""
        for it in items:
            if it["t"] == "stmt":
                target = it["target"] if it["role"] == "init" else ops[str(it["op"])]["result"]
                if st[target]["cls"] != "contracted":
                    acc["steps"] += trips * m.stmt_us
                continue
            rng = ext[it["extent"]] / nb if it["sliced"] else ext[it["extent"]]
            if has_loop(it["body"]):
                walk(it["body"], trips * max(rng, 1.0), nb, threads, acc)
                continue
            # strided (innermost) loop
            per_thread = max(1.0, rng / threads)
            mats, vecs, rmw = set(), set(), False
            for s in it["body"]:
                if s["role"] == "init":
                    names, target, red = [s["target"]], s["target"], False
                else:
                    op = ops[str(s["op"])]
                    names, target, red = list(op["operands"]) + [op["result"]], op["result"], op["reduction"]
                    if red and it["axis"] in st[target]["labels"] and st[target]["cls"] != "contracted":
                        rmw = True
                for n in names:
                    s_ = st[n]
                    if s_["cls"] == "contracted" or it["axis"] not in s_["labels"]:
                        continue
                    (mats if len(s_["labels"]) == 2 else vecs).add(n)
            acc["bytes"] += 8.0 * len(mats) * rng * trips * nb + 8.0 * len(vecs) * rng * nb
            acc["steps"] += trips * (m.step_us + per_thread * (m.rmw_trip_us if rmw else m.trip_us))

    def close(acc, nb):
        bw = min(m.peak_gbs, m.cta_gbs * min(nb, 4 * m.sm_count)) * 1e9
        per_launch.append((m.launch_us + max(acc["bytes"] / bw * 1e6, acc["steps"])) * 1e-6)

    serial = None
    for root in ir["roots"]:
        if root["t"] != "par":
            if serial is None:
                serial = {"bytes": 0.0, "steps": 0.0}
                launches += 1
            walk([root], 1.0, 1.0, float(SERIAL_THREADS), serial)
            continue
        if serial is not None:
            close(serial, 1.0)
            serial = None
        org_t = float(ir["threads"][root["slot"]])
        nb = max(org_t, float(blocks))
        em = _Emitter(ir, blocks)
        if em.has_sliced_lane_loop(root["body"]):
            nb = min(nb, max(org_t, float(int(ext[root["extent"]]) // CTA_THREADS)))
        nb = max(1.0, min(nb, ext[root["extent"]]))
        acc = {"bytes": 0.0, "steps": 0.0}
        walk(root["body"], 1.0, nb, float(CTA_THREADS), acc)
        close(acc, nb)
        launches += 1
        for result in root["partials"]:          # join: read nb partial rows, write the result
            p = st[em.partial_for(result)]
            size = 1.0
            for e in p["extents"]:
                size *= ext[e]
            per_launch.append((m.launch_us + 8.0 * size * (nb + 1) / (m.peak_gbs * 1e9) * 1e6
                               + (nb * 0.01 if not p["extents"] else 0.0)) * 1e-6)
            launches += 1
    if serial is not None:
        close(serial, 1.0)
    nalloc = sum(1 for s in st.values() if s["cls"] in ("temp", "partial"))
    per_launch.append(nalloc * m.alloc_us * 1e-6)
    contracted = tuple(sorted(n for n, s in st.items() if s["cls"] == "contracted"))
    return CostReport(total=float(sum(per_launch)), source="analytic", per_root=tuple(per_launch),
                      contracted=contracted, partition_nodes=launches)


class AnalyticOrganismCost:
    """Fitness callable over the reference's Organism objects (cost.py:106-121 with
    the GPU model): organism -> lower -> contract_arrays -> estimate_cost_ir."""

    parallel_safe = True

    def __init__(self, ref_graph, extents: dict, model: EmitModel | None = None,
                 blocks: int = DEFAULT_BLOCKS):
        self.ref_graph, self.extents, self.model, self.blocks = ref_graph, dict(extents), model, blocks

    def key_salt(self) -> str:
        return "analytic-cuda:" + ",".join(f"{k}={v}" for k, v in sorted(self.extents.items()))

    def __call__(self, organism):
        from matfuse import contract_arrays, lower
        ir = ir_from_matfuse(contract_arrays(lower(organism, self.ref_graph)))
        return estimate_cost_ir(ir, self.extents, self.model, self.blocks)
