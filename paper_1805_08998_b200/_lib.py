"""ctypes binding of ``libhx.so`` (the C ABI declared in ``include/hx.h``).

The library is built in-tree by ``paper_1805_08998_b200/build.py`` (called from
``__graft_entry__.build()``).  There is no fallback: if the library is missing every entry
point raises, so a product call can never silently run on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HX_LIB", os.path.join(HERE, "libhx.so"))

i8p = C.POINTER(C.c_int8)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class HxTree(C.Structure):
    _fields_ = [("n_clusters", C.c_int32), ("c_lo", i64p), ("c_hi", i64p),
                ("c_child", i32p), ("n_nodes", C.c_int32), ("tau", i32p), ("sigma", i32p),
                ("kind", i8p), ("child", i32p)]


class HxOperand(C.Structure):
    _fields_ = [("payload", i8p), ("rank", i32p), ("u_off", i64p), ("v_off", i64p),
                ("d_off", i64p)]


class HxPlanInfo(C.Structure):
    _fields_ = [(name, C.c_int64) for name in (
        "n_out", "n_far", "n_near", "n_terms_real", "n_terms_expand", "n_dxd")] + [
        ("created", C.c_int64 * 3)] + [(name, C.c_int64) for name in (
            "mat_terms", "mat_tiles", "mat_groups", "core_terms", "core_tiles", "fac_terms",
            "fac_tiles", "core_elems", "term_elems", "tile_elems", "max_out_dim",
            "n_xgroups", "gather_elems", "gather_jobs")] + [
        (name, C.c_double) for name in ("flops_form", "bytes_form", "flops_near",
                                        "bytes_near")]


class HxProductCfg(C.Structure):
    _fields_ = [("policy", C.c_int32), ("eps", C.c_double), ("k_max", C.c_int32),
                ("tag", C.c_int32), ("seed", C.c_uint64), ("sketch0", C.c_int32),
                ("oversample", C.c_int32), ("q", C.c_int32)]


class HxProductStats(C.Structure):
    _fields_ = [(name, C.c_double) for name in ("ms_total", "ms_form", "ms_mat",
                                                "ms_recompress")] + [
        (name, C.c_int64) for name in ("far_leaves", "near_leaves", "degraded_blocks",
                                       "max_far_rank", "matvec_count", "sketch_rounds",
                                       "launches", "out_elems")] + [
        ("fro2_total", C.c_double), ("dom_kernel_ms", C.c_double), ("ms_upload", C.c_double),
        ("t_marks", C.c_double * 4), ("sketch_cols", C.c_int64)]


class HxError(RuntimeError):
    pass


_lib = None

SIGNATURES = {
    "hx_plan_create": [C.POINTER(HxTree), C.POINTER(HxOperand), C.POINTER(HxOperand), u8p,
                       C.c_int, C.c_int, C.POINTER(C.c_void_p)],
    "hx_plan_info_get": [C.c_void_p, C.POINTER(HxPlanInfo)],
    "hx_plan_leaves": [C.c_void_p, i32p, i8p, i32p, i32p, i64p, f64p, f64p],
    "hx_plan_term_log": [C.c_void_p, i32p, i8p, i32p, i32p, i32p],
    "hx_plan_free": [C.c_void_p],
    "hx_plan_mma_flops": [C.c_void_p, f64p],
    "hx_ctx_create": [C.c_int, C.POINTER(C.c_void_p)],
    "hx_ctx_operand": [C.c_void_p, C.c_int, f64p, C.c_void_p, C.c_int64],
    "hx_ctx_operand_alias": [C.c_void_p],
    "hx_product": [C.c_void_p, C.c_void_p, C.POINTER(HxProductCfg),
                   C.POINTER(HxProductStats)],
    "hx_result_layout": [C.c_void_p, i32p, i8p, i64p],
    "hx_result_download": [C.c_void_p, f64p, C.c_int64],
    "hx_assemble": [C.c_void_p, C.POINTER(HxTree), f64p, C.c_int, C.c_int, C.c_double,
                    C.c_double, i8p, i32p, i64p, i64p, i64p, i8p, C.POINTER(C.c_void_p), i64p],
    "hx_pool_download": [C.c_void_p, C.c_void_p, f64p, C.c_int64],
    "hx_pool_free": [C.c_void_p, C.c_void_p],
    "hx_ctx_synchronize": [C.c_void_p],
    "hx_ctx_mem_info": [C.c_void_p, i64p, i64p],
    "hx_ctx_trim": [C.c_void_p],
    "hx_ctx_reset_hints": [C.c_void_p],
    "hx_ctx_operand_share": [C.c_void_p, C.c_void_p],
    "hx_ctx_held_bytes": [C.c_void_p],
    "hx_timeline_epoch": [],
    "hx_host_alloc": [C.c_int64],
    "hx_host_free": [C.c_void_p, C.c_int64],
    "hx_host_register": [C.c_void_p, C.c_int64],
    "hx_host_unregister": [C.c_void_p],
    "hx_operand_layout": [C.POINTER(HxTree), i8p, i32p, i64p, i64p, i64p, i64p],
    "hx_hmx1_write": [C.c_char_p, C.POINTER(HxTree), C.c_int64, u8p, C.POINTER(HxOperand),
                      i8p, f64p],
    "hx_hmx1_scan": [C.c_char_p, C.POINTER(HxTree), C.c_int64, u8p, i8p, i32p, i8p, i64p],
    "hx_hmx1_read": [C.c_char_p, C.POINTER(HxTree), C.POINTER(HxOperand), i64p, f64p],
    "hx_hmatvec": [C.c_void_p, C.POINTER(HxTree), C.POINTER(HxOperand), C.c_int, C.c_int,
                   f64p, f64p, C.c_int],
    "hx_debug_gemm": [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                      C.c_int64, C.POINTER(f64p), i64p, f64p, C.c_int64],
    "hx_debug_qr": [C.c_int, i32p, i32p, f64p, f64p],
    "hx_np_normals": [C.c_uint64, C.c_uint64, C.c_int64, f64p, C.c_int],
    "hx_debug_compress": [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_int32,
                          C.c_int, C.c_int, f64p, f64p, f64p, i32p],
    "hx_ctx_free": [C.c_void_p],
    "hx_last_error": [C.c_char_p, C.c_size_t],
    "hx_version": [],
}
VOID_RET = {"hx_plan_free", "hx_ctx_free", "hx_host_free"}
INT64_RET = {"hx_ctx_held_bytes"}
PTR_RET = {"hx_host_alloc"}

STATUS_EXC = {-1: ValueError, -2: MemoryError, -3: HxError, -4: NotImplementedError}


def lib():
    """The loaded library; raises if it was not built (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HxError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            if not hasattr(L, name):   # partial test builds (planner only)
                continue
            f = getattr(L, name)
            f.argtypes = args
            f.restype = None if name in VOID_RET else (
                C.c_int64 if name in INT64_RET else (C.c_void_p if name in PTR_RET else C.c_int))
        _lib = L
        _tune_host_allocator()
    return _lib


def _tune_host_allocator():
    """Opt-in (HX_MALLOPT=1, set by bench.py): keep freed heap memory in the process (glibc
    mallopt).  The per-product work lists (tens of MB of std::vector, rebuilt every product)
    otherwise go back to the kernel with munmap / trim and come back as fresh page faults,
    which showed up as 40-90 ms stalls on some products (config 2: mean step 331 -> 319 ms,
    worst of 39 steps 414 -> 351 ms).  It changes the allocator of the whole process, so a
    library user has to ask for it."""
    if os.environ.get("HX_MALLOPT", "0") in ("", "0"):
        return
    try:
        libc = C.CDLL("libc.so.6")
        M_TRIM_THRESHOLD, M_TOP_PAD, M_MMAP_THRESHOLD = -1, -2, -3
        libc.mallopt(M_MMAP_THRESHOLD, 32 << 20)   # the largest threshold glibc accepts
        libc.mallopt(M_TRIM_THRESHOLD, (1 << 31) - 1)
        libc.mallopt(M_TOP_PAD, 512 << 20)
    except OSError:  # pragma: no cover - not glibc
        pass


def last_error():
    buf = C.create_string_buffer(4096)
    lib().hx_last_error(buf, 4096)
    return buf.value.decode(errors="replace")


def check(code, what):
    if code != 0:
        exc = STATUS_EXC.get(code, HxError)
        raise exc(f"{what}: {last_error()}")


def ptr(a, typ):
    if a is None:
        return None
    return a.ctypes.data_as(typ)


class TreeBuf:
    """Keeps the numpy arrays behind an ``hx_tree`` alive."""

    def __init__(self, arrays):
        self.arrays = arrays
        a = arrays
        self.st = HxTree(len(a["c_lo"]), ptr(a["c_lo"], i64p), ptr(a["c_hi"], i64p),
                         ptr(a["c_child"], i32p), len(a["tau"]), ptr(a["tau"], i32p),
                         ptr(a["sigma"], i32p), ptr(a["kind"], i8p), ptr(a["child"], i32p))


class OperandBuf:
    def __init__(self, d):
        self.d = {k: np.ascontiguousarray(v) for k, v in d.items()}
        x = self.d
        self.st = HxOperand(ptr(x["payload"], i8p), ptr(x["rank"], i32p), ptr(x["u_off"], i64p),
                            ptr(x["v_off"], i64p), ptr(x["d_off"], i64p))


class Plan:
    """Owning wrapper of an ``hx_plan``."""

    DEFER = 1  # HX_PLAN_DEFER: factor work lists filled by hx_product, batch by batch
    LOG = 2    # HX_PLAN_LOG: keep the restrict log (term_log)

    def __init__(self, tree_arrays, opa, opb, leaf_mask=None, tile=64, flags=0):
        self.tree = TreeBuf(tree_arrays)
        self.opa = OperandBuf(opa)
        self.opb = self.opa if opb is opa else OperandBuf(opb)
        self.mask = None if leaf_mask is None else np.ascontiguousarray(leaf_mask, np.uint8)
        h = C.c_void_p()
        check(lib().hx_plan_create(C.byref(self.tree.st), C.byref(self.opa.st),
                                   C.byref(self.opb.st), ptr(self.mask, u8p), tile, flags,
                                   C.byref(h)), "hx_plan_create")
        self.h = h
        self.info = HxPlanInfo()
        check(lib().hx_plan_info_get(self.h, C.byref(self.info)), "hx_plan_info_get")

    def leaves(self):
        n = self.info.n_out
        ids = np.zeros(n, np.int32)
        kind = np.zeros(n, np.int8)
        m = np.zeros(n, np.int32)
        nn = np.zeros(n, np.int32)
        K = np.zeros(n, np.int64)
        fdd = np.zeros(n)
        edd = np.zeros(n)
        check(lib().hx_plan_leaves(self.h, ptr(ids, i32p), ptr(kind, i8p), ptr(m, i32p),
                                   ptr(nn, i32p), ptr(K, i64p), ptr(fdd, f64p),
                                   ptr(edd, f64p)), "hx_plan_leaves")
        return dict(ids=ids, kind=kind, m=m, n=nn, K=K, fdd=fdd, edd=edd)

    def term_log(self):
        n = self.info.n_terms_real
        out = dict(block=np.zeros(n, np.int32), kind=np.zeros(n, np.int8),
                   a=np.zeros(n, np.int32), b=np.zeros(n, np.int32), rank=np.zeros(n, np.int32))
        check(lib().hx_plan_term_log(self.h, ptr(out["block"], i32p), ptr(out["kind"], i8p),
                                     ptr(out["a"], i32p), ptr(out["b"], i32p),
                                     ptr(out["rank"], i32p)), "hx_plan_term_log")
        return out

    def close(self):
        if self.h:
            lib().hx_plan_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


def pinned_empty(n, dtype=np.float64):
    """numpy array of n elements in page-locked memory from the library's cache (returned to
    the cache when the array and every view of it are gone)."""
    import weakref
    itemsize = np.dtype(dtype).itemsize
    nbytes = max(int(n), 1) * itemsize
    p = lib().hx_host_alloc(nbytes)
    if not p:
        raise MemoryError("hx_host_alloc failed")
    buf = (C.c_char * nbytes).from_address(p)
    arr = np.frombuffer(buf, dtype=dtype, count=max(int(n), 1))
    weakref.finalize(buf, lib().hx_host_free, p, nbytes)
    return arr


def pin_host_array(a):
    """Page-lock a caller-owned array in place (uploads become DMA); undone when it dies."""
    import weakref
    if a.nbytes == 0 or getattr(a, "_hx_pinned", False):
        return
    p = a.ctypes.data
    if lib().hx_host_register(C.c_void_p(p), a.nbytes) == 0:
        weakref.finalize(a, lib().hx_host_unregister, C.c_void_p(p))
