"""Text formats and host-side data preparation, reference-shaped.

Mirrors include/cmtf/sparse_data.hpp:86-112 (load_tensor, load_matrix,
save_tensor, save_matrix, split_train_test) and include/cmtf/model_io.hpp
(save_model, load_model) over the C ABI (csrc/io.cpp: multi-threaded parse
and formatting; the SparseTensor / CoupledMatrix constructor checks --
check_entries, src/sparse_data.cpp:19-64 -- run on the device through
cmtf_gpu_check_entries).  Same error types and messages as the reference:
ParseError for malformed files, ValidationError for bad entries.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .api import (CmtfError, CoupledMatrix, FactorModel, ParseError, SparseTensor,
                  ValidationError, _ptr, _raise)


def _fail(rc: int):
    msg = _abi.lib().cmtf_gpu_last_error().decode()
    if rc == _abi.EPARSE:
        raise ParseError(msg)
    _raise(rc, msg)


def _parse(path, expected_order: int, threads: int):
    L = _abi.lib()
    h = C.c_void_p()
    rc = L.cmtf_coo_parse(os.fsencode(str(path)), expected_order, threads, C.byref(h))
    if rc:
        _fail(rc)
    try:
        order = L.cmtf_coo_order(h)
        nnz = L.cmtf_coo_nnz(h)
        dims = np.ctypeslib.as_array(L.cmtf_coo_dims(h), (order,)).copy()
        if nnz:
            idx = np.ctypeslib.as_array(L.cmtf_coo_indices(h), (nnz * order,)).copy()
            vals = np.ctypeslib.as_array(L.cmtf_coo_values(h), (nnz,)).copy()
        else:
            idx = np.zeros(0, np.uint32)
            vals = np.zeros(0)
        return order, bool(L.cmtf_coo_has_header(h)), [int(d) for d in dims], \
            idx.reshape(nnz, order), vals
    finally:
        L.cmtf_coo_free(h)


def check_entries(dims: Sequence[int], indices, values, is_matrix: bool = False,
                  device: int = 0):
    """check_entries (src/sparse_data.cpp:19-64) on the device."""
    dims = np.ascontiguousarray(dims, dtype=np.uint32)
    indices = np.ascontiguousarray(indices, dtype=np.uint32)
    values = np.ascontiguousarray(values, dtype=np.float64)
    rc = _abi.lib().cmtf_gpu_check_entries(device, len(dims), _ptr(dims, C.c_uint32),
                                           _ptr(indices, C.c_uint32),
                                           _ptr(values, C.c_double), values.shape[0],
                                           int(is_matrix))
    if rc:
        _fail(rc)


def load_tensor(path, threads: int = 0, check: bool = True, device: int = 0) -> SparseTensor:
    """load_tensor (src/sparse_data.cpp:247-254): parse, infer dims, then the
    SparseTensor constructor's validation (on the device; check=False skips
    it, e.g. on a host without a GPU)."""
    order, _, dims, idx, vals = _parse(path, 0, threads)
    if order + 1 < 3:
        raise ParseError(f"'{path}': tensor order must be at least 2")
    if check:
        check_entries(dims, idx, vals, False, device)
    return SparseTensor(dims, idx, vals)


def load_matrix(path, coupled_mode: int, weight: float, tensor: SparseTensor,
                threads: int = 0, check: bool = True, device: int = 0) -> CoupledMatrix:
    """load_matrix (src/sparse_data.cpp:256-277); coupled_mode is 1-based as
    on the command line."""
    if coupled_mode < 1 or coupled_mode > tensor.order:
        raise ValidationError(f"coupled mode {coupled_mode} out of range 1..{tensor.order}")
    if not weight > 0:
        raise ValidationError("lambda_m must be positive")
    _, header, dims, idx, vals = _parse(path, 2, threads)
    rows = tensor.dims[coupled_mode - 1]
    if header and dims[0] != rows:
        raise ValidationError(f"'{path}': matrix has {dims[0]} rows but mode {coupled_mode} "
                              f"has size {rows}")
    if dims[0] > rows:
        raise ValidationError(f"'{path}': matrix row index exceeds size of mode {coupled_mode}")
    if check:
        check_entries([rows, dims[1]], idx, vals, True, device)
    return CoupledMatrix(coupled_mode - 1, rows, dims[1], idx, vals, weight)


def _write(path, dims, idx, vals, threads):
    dims = np.ascontiguousarray(dims, dtype=np.uint32)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    rc = _abi.lib().cmtf_coo_write(os.fsencode(str(path)), len(dims), _ptr(dims, C.c_uint32),
                                   _ptr(idx, C.c_uint32), _ptr(vals, C.c_double),
                                   vals.shape[0], threads)
    if rc:
        _fail(rc)


def save_tensor(path, t: SparseTensor, threads: int = 0):
    """save_tensor (src/sparse_data.cpp:304-306)."""
    _write(path, t.dims, t.indices, t.values, threads)


def save_matrix(path, m: CoupledMatrix, threads: int = 0):
    """save_matrix (src/sparse_data.cpp:308-311)."""
    _write(path, [m.rows, m.cols], m.indices, m.values, threads)


def split_train_test(t: SparseTensor, test_fraction: float, seed: int,
                     threads: int = 0) -> Tuple[SparseTensor, SparseTensor]:
    """split_train_test (src/sparse_data.cpp:311-342) -> (train, test)."""
    L = _abi.lib()
    idx = np.ascontiguousarray(t.indices, dtype=np.uint32)
    vals = np.ascontiguousarray(t.values, dtype=np.float64)
    nt = C.c_uint64()
    null_u, null_f = C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)()
    rc = L.cmtf_split_train_test(t.order, _ptr(idx, C.c_uint32), _ptr(vals, C.c_double), t.nnz,
                                 test_fraction, seed, null_u, null_f, null_u, null_f,
                                 C.byref(nt), threads)
    if rc:
        _fail(rc)
    n_test = nt.value
    tr_i = np.zeros((t.nnz - n_test, t.order), np.uint32)
    tr_v = np.zeros(t.nnz - n_test)
    te_i = np.zeros((n_test, t.order), np.uint32)
    te_v = np.zeros(n_test)
    rc = L.cmtf_split_train_test(t.order, _ptr(idx, C.c_uint32), _ptr(vals, C.c_double), t.nnz,
                                 test_fraction, seed, _ptr(tr_i, C.c_uint32),
                                 _ptr(tr_v, C.c_double), _ptr(te_i, C.c_uint32),
                                 _ptr(te_v, C.c_double), C.byref(nt), threads)
    if rc:
        _fail(rc)
    return SparseTensor(t.dims, tr_i, tr_v), SparseTensor(t.dims, te_i, te_v)


def save_model(path, model: FactorModel, coupling_modes: Optional[Sequence[int]] = None,
               cp: bool = False):
    """save_model (src/model_io.cpp:94-126).  coupling_modes: 0-based mode of
    each coupled factor (default: model.coupling_modes).  cp: model.core
    holds the CP superdiagonal (ranks[0] values) instead of the dense core."""
    L = _abi.lib()
    ranks = np.ascontiguousarray([f.shape[1] for f in model.factors], dtype=np.uint32)
    core = np.ascontiguousarray(model.core, dtype=np.float64).reshape(-1)
    facs = [np.ascontiguousarray(f, dtype=np.float64) for f in model.factors]
    rows = np.ascontiguousarray([f.shape[0] for f in facs], dtype=np.uint32)
    fp = (C.POINTER(C.c_double) * len(facs))(*[_ptr(f, C.c_double) for f in facs])
    modes = list(coupling_modes if coupling_modes is not None
                 else getattr(model, "coupling_modes", []) or [])
    cps = [np.ascontiguousarray(c, dtype=np.float64) for c in model.couplings]
    if len(modes) != len(cps):
        raise ValidationError("one coupled mode per coupled factor is needed")
    cm = np.ascontiguousarray(modes, dtype=np.int32)
    cr = np.ascontiguousarray([c.shape[0] for c in cps], dtype=np.uint32)
    cpp = (C.POINTER(C.c_double) * max(1, len(cps)))(*[_ptr(c, C.c_double) for c in cps])
    rc = L.cmtf_model_save(os.fsencode(str(path)), len(ranks), _ptr(ranks, C.c_uint32), int(cp),
                           _ptr(core, C.c_double), _ptr(rows, C.c_uint32), fp, len(cps),
                           _ptr(cm, C.c_int32), _ptr(cr, C.c_uint32), cpp)
    if rc:
        _fail(rc)


def load_model(path) -> FactorModel:
    """load_model (src/model_io.cpp:128-179); the core comes back dense, the
    coupled factors' modes in model.coupling_modes."""
    L = _abi.lib()
    h = C.c_void_p()
    rc = L.cmtf_model_load(os.fsencode(str(path)), C.byref(h))
    if rc:
        _fail(rc)
    try:
        order = L.cmtf_model_order(h)
        ranks = [int(r) for r in np.ctypeslib.as_array(L.cmtf_model_ranks(h), (order,))]
        core = np.ctypeslib.as_array(L.cmtf_model_core(h), (int(np.prod(ranks)),)).copy()
        facs = []
        for n in range(order):
            r = L.cmtf_model_factor_rows(h, n)
            facs.append(np.ctypeslib.as_array(L.cmtf_model_factor(h, n),
                                              (r * ranks[n],)).copy().reshape(r, ranks[n]))
        cps, modes = [], []
        for c in range(L.cmtf_model_n_coupled(h)):
            mode = L.cmtf_model_coupled_mode(h, c)
            r = L.cmtf_model_coupled_rows(h, c)
            cps.append(np.ctypeslib.as_array(L.cmtf_model_coupled(h, c),
                                             (r * ranks[mode],)).copy().reshape(r, ranks[mode]))
            modes.append(mode)
    finally:
        L.cmtf_model_free(h)
    m = FactorModel(core.reshape(ranks), facs, cps)
    m.coupling_modes = modes
    return m
