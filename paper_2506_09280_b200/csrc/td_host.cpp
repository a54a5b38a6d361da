// _td_host: the per-record walks of a warm check() (plan-cache hit) in C++.
//
// A cached plan is reused when the new traces have the same layout, and it
// is bound to their payloads by record position (checker._check_direct).
// Both steps walk every record: the layout key (ids, rank metas, mapping
// signature ids, dtypes, shapes, replica sizes; checker._layout_key) and the
// operand pointers (device._resolve_resident), plus the host-bytes scan that
// decides whether anything must be staged.  In Python each walk costs
// ~0.3-0.5 us per record in torch attribute getters (is_cuda, dtype, shape,
// is_contiguous, data_ptr); here the payload is unpacked once to its
// at::Tensor and read directly.
//
// Every function returns exactly what its Python counterpart returns (the
// Python path stays as the fallback and the tests compare the two), or None
// to hand a case it does not cover back to Python.  Host metadata only: no
// payload byte is read here.
#include <Python.h>

#include <torch/csrc/autograd/python_variable.h>

#include <cstdint>
#include <cstring>

namespace {

PyObject* s_payload;
PyObject* s_id;
PyObject* s_encode;
PyObject* s_rank_meta;
PyObject* s_as_tuple;
PyObject* s_mapping;
PyObject* s_sig_id;
PyObject* s_replica;
PyObject* s_dtype_code;
PyObject* s_text;
PyObject* s_t;

// td dtype code of a tensor (td_api.h TD_F32/BF16/F16/F64), -1 otherwise
int td_code(const at::Tensor& t) {
    switch (t.scalar_type()) {
        case at::kFloat: return 0;
        case at::kBFloat16: return 1;
        case at::kHalf: return 2;
        case at::kDouble: return 3;
        default: return -1;
    }
}

struct Seq {
    PyObject* fast = nullptr;
    Py_ssize_t n = 0;
    PyObject** items = nullptr;
    explicit Seq(PyObject* o) {
        fast = PySequence_Fast(o, "expected a sequence");
        if (fast) {
            n = PySequence_Fast_GET_SIZE(fast);
            items = PySequence_Fast_ITEMS(fast);
        }
    }
    ~Seq() { Py_XDECREF(fast); }
};

// obj.<cache> when the immutable object already memoised it (CanonicalId
// keeps its encoded text in _text, RankMeta its tuple in _t), else
// obj.<method>(), which memoises it: no Python frame on the warm path.
PyObject* cached_or_call(PyObject* obj, PyObject* cache, PyObject* method) {
    PyObject* v = PyObject_GetAttr(obj, cache);
    if (v) return v;
    if (!PyErr_ExceptionMatches(PyExc_AttributeError)) return nullptr;
    PyErr_Clear();
    return PyObject_CallMethodNoArgs(obj, method);
}

// layout_key(records) -> (ids, rank tuples, signature ids, dtype codes,
// shapes, replica sizes): six tuples in record order, equal to
// checker._layout_key's (torch.Size compares and hashes as its tuple).
PyObject* layout_key(PyObject*, PyObject* arg) {
    Seq recs(arg);
    if (!recs.fast) return nullptr;
    const Py_ssize_t n = recs.n;
    PyObject* cols[6];
    for (auto& c : cols) c = PyTuple_New(n);
    bool ok = cols[0] && cols[1] && cols[2] && cols[3] && cols[4] && cols[5];
    for (Py_ssize_t k = 0; ok && k < n; ++k) {
        PyObject* rec = recs.items[k];
        PyObject* id = PyObject_GetAttr(rec, s_id);
        PyObject* enc = id ? cached_or_call(id, s_text, s_encode) : nullptr;
        Py_XDECREF(id);
        PyObject* rm = PyObject_GetAttr(rec, s_rank_meta);
        PyObject* rt = rm ? cached_or_call(rm, s_t, s_as_tuple) : nullptr;
        Py_XDECREF(rm);
        PyObject* mp = PyObject_GetAttr(rec, s_mapping);
        PyObject* sig = mp ? PyObject_GetAttr(mp, s_sig_id) : nullptr;
        Py_XDECREF(mp);
        PyObject* rep = PyObject_GetAttr(rec, s_replica);
        PyObject* payload = PyObject_GetAttr(rec, s_payload);
        PyObject* code = nullptr;
        PyObject* shape = nullptr;
        if (payload && THPVariable_Check(payload)) {
            const at::Tensor& t = THPVariable_Unpack(payload);
            const int c = td_code(t);
            code = c >= 0 ? PyLong_FromLong(c) : PyObject_GetAttr(rec, s_dtype_code);   // raises as Python does
            const auto sizes = t.sizes();
            shape = PyTuple_New((Py_ssize_t)sizes.size());
            for (size_t a = 0; shape && a < sizes.size(); ++a)
                PyTuple_SET_ITEM(shape, (Py_ssize_t)a, PyLong_FromLongLong(sizes[a]));
        } else if (payload) {
            code = PyObject_GetAttr(rec, s_dtype_code);
            PyObject* sh = PyObject_GetAttrString(payload, "shape");
            shape = sh ? PySequence_Tuple(sh) : nullptr;
            Py_XDECREF(sh);
        }
        Py_XDECREF(payload);
        if (!(enc && rt && sig && rep && code && shape)) {
            Py_XDECREF(enc); Py_XDECREF(rt); Py_XDECREF(sig); Py_XDECREF(rep); Py_XDECREF(code); Py_XDECREF(shape);
            ok = false;
            break;
        }
        PyTuple_SET_ITEM(cols[0], k, enc);
        PyTuple_SET_ITEM(cols[1], k, rt);
        PyTuple_SET_ITEM(cols[2], k, sig);
        PyTuple_SET_ITEM(cols[3], k, code);
        PyTuple_SET_ITEM(cols[4], k, shape);
        PyTuple_SET_ITEM(cols[5], k, rep);
    }
    if (!ok) {
        for (auto& c : cols) Py_XDECREF(c);
        return nullptr;
    }
    PyObject* res = PyTuple_Pack(6, cols[0], cols[1], cols[2], cols[3], cols[4], cols[5]);
    for (auto& c : cols) Py_DECREF(c);
    return res;
}

// td dtype code of a record's payload as a new int (rec.dtype_code's value;
// non-torch payloads and unsupported dtypes go through the property, which
// raises as Python does)
PyObject* record_code(PyObject* rec, PyObject* payload) {
    if (THPVariable_Check(payload)) {
        const int c = td_code(THPVariable_Unpack(payload));
        if (c >= 0) return PyLong_FromLong(c);
    }
    return PyObject_GetAttr(rec, s_dtype_code);
}

// group_by_id(records) -> (ids, positions, keys): the encoded ids in first
// appearance order (Trace.by_id's order), each id's record positions in
// trace order, and each id's merge_view structure key — the tuple of
// (mapping signature id, replica group size, dtype code) of its records.
PyObject* group_by_id(PyObject*, PyObject* arg) {
    Seq recs(arg);
    if (!recs.fast) return nullptr;
    PyObject* index = PyDict_New();
    PyObject* ids = PyList_New(0);
    PyObject* pos = PyList_New(0);
    PyObject* atoms = PyList_New(0);
    bool ok = index && ids && pos && atoms;
    for (Py_ssize_t k = 0; ok && k < recs.n; ++k) {
        PyObject* rec = recs.items[k];
        PyObject* id = PyObject_GetAttr(rec, s_id);
        PyObject* enc = id ? cached_or_call(id, s_text, s_encode) : nullptr;
        Py_XDECREF(id);
        PyObject* mp = enc ? PyObject_GetAttr(rec, s_mapping) : nullptr;
        PyObject* sig = mp ? PyObject_GetAttr(mp, s_sig_id) : nullptr;
        Py_XDECREF(mp);
        PyObject* rep = sig ? PyObject_GetAttr(rec, s_replica) : nullptr;
        PyObject* payload = rep ? PyObject_GetAttr(rec, s_payload) : nullptr;
        PyObject* code = payload ? record_code(rec, payload) : nullptr;
        Py_XDECREF(payload);
        PyObject* atom = code ? PyTuple_Pack(3, sig, rep, code) : nullptr;
        Py_XDECREF(sig); Py_XDECREF(rep); Py_XDECREF(code);
        PyObject* kk = atom ? PyLong_FromSsize_t(k) : nullptr;
        if (!kk) {
            Py_XDECREF(enc); Py_XDECREF(atom);
            ok = false;
            break;
        }
        PyObject* slot = PyDict_GetItemWithError(index, enc);     // borrowed
        if (slot) {
            const Py_ssize_t j = PyLong_AsSsize_t(slot);
            ok = PyList_Append(PyList_GET_ITEM(pos, j), kk) == 0 &&
                 PyList_Append(PyList_GET_ITEM(atoms, j), atom) == 0;
        } else if (!PyErr_Occurred()) {
            PyObject* j = PyLong_FromSsize_t(PyList_GET_SIZE(ids));
            PyObject* pl = PyList_New(1);
            PyObject* al = PyList_New(1);
            ok = j && pl && al && PyDict_SetItem(index, enc, j) == 0 && PyList_Append(ids, enc) == 0;
            if (ok) {
                Py_INCREF(kk); PyList_SET_ITEM(pl, 0, kk);
                Py_INCREF(atom); PyList_SET_ITEM(al, 0, atom);
                ok = PyList_Append(pos, pl) == 0 && PyList_Append(atoms, al) == 0;
            }
            Py_XDECREF(j); Py_XDECREF(pl); Py_XDECREF(al);
        } else {
            ok = false;
        }
        Py_DECREF(enc); Py_DECREF(atom); Py_DECREF(kk);
    }
    PyObject* keys = ok ? PyList_New(PyList_GET_SIZE(atoms)) : nullptr;
    for (Py_ssize_t j = 0; keys && j < PyList_GET_SIZE(atoms); ++j) {
        PyObject* t = PyList_AsTuple(PyList_GET_ITEM(atoms, j));
        if (!t) {
            Py_CLEAR(keys);
            break;
        }
        PyList_SET_ITEM(keys, j, t);
    }
    PyObject* res = keys ? PyTuple_Pack(3, ids, pos, keys) : nullptr;
    Py_XDECREF(index); Py_XDECREF(ids); Py_XDECREF(pos); Py_XDECREF(atoms); Py_XDECREF(keys);
    return res;
}

// host_bytes(records) -> bytes of payloads not resident on a CUDA device
// (checker._host_bytes), or None when a payload is not a torch tensor (numpy
// payloads: the Python walk sums record.nbytes).
PyObject* host_bytes(PyObject*, PyObject* arg) {
    Seq recs(arg);
    if (!recs.fast) return nullptr;
    long long total = 0;
    for (Py_ssize_t k = 0; k < recs.n; ++k) {
        PyObject* payload = PyObject_GetAttr(recs.items[k], s_payload);
        if (!payload) return nullptr;
        if (!THPVariable_Check(payload)) {
            Py_DECREF(payload);
            Py_RETURN_NONE;
        }
        const at::Tensor& t = THPVariable_Unpack(payload);
        if (!t.is_cuda()) total += (long long)(t.numel() * t.element_size());
        Py_DECREF(payload);
    }
    return PyLong_FromLongLong(total);
}

// resident_ptrs(operands, want) -> (pointer bytes (u64 per operand), payload
// list) when every operand is a record whose payload is a contiguous CUDA
// tensor of td dtype want[k] at a 16-byte aligned address; None otherwise
// (device._resolve_resident's contract).  want: bytes, one code per operand.
PyObject* resident_ptrs(PyObject*, PyObject* args) {
    PyObject* ops_obj;
    Py_buffer want;
    if (!PyArg_ParseTuple(args, "Oy*", &ops_obj, &want)) return nullptr;
    Seq ops(ops_obj);
    if (!ops.fast) {
        PyBuffer_Release(&want);
        return nullptr;
    }
    if (want.len != ops.n) {
        PyBuffer_Release(&want);
        PyErr_SetString(PyExc_ValueError, "resident_ptrs: one dtype code per operand");
        return nullptr;
    }
    const unsigned char* w = static_cast<const unsigned char*>(want.buf);
    PyObject* ptrs = PyBytes_FromStringAndSize(nullptr, ops.n * (Py_ssize_t)sizeof(uint64_t));
    PyObject* keep = PyList_New(ops.n);
    if (!ptrs || !keep) {
        Py_XDECREF(ptrs); Py_XDECREF(keep);
        PyBuffer_Release(&want);
        return nullptr;
    }
    uint64_t* out = reinterpret_cast<uint64_t*>(PyBytes_AS_STRING(ptrs));
    bool fast = true;
    for (Py_ssize_t k = 0; fast && k < ops.n; ++k) {
        PyObject* payload = PyObject_GetAttr(ops.items[k], s_payload);
        if (!payload) {          // not a record (a raw operand): general path
            PyErr_Clear();
            fast = false;
            break;
        }
        if (THPVariable_Check(payload)) {
            const at::Tensor& t = THPVariable_Unpack(payload);
            if (t.is_cuda() && td_code(t) == (int)w[k] && t.is_contiguous()) {
                const uint64_t p = (uint64_t)(uintptr_t)t.data_ptr();
                if ((p & 15u) == 0) {
                    out[k] = p;
                    PyList_SET_ITEM(keep, k, payload);   // steals the reference
                    continue;
                }
            }
        }
        Py_DECREF(payload);
        fast = false;
    }
    PyBuffer_Release(&want);
    if (!fast) {
        Py_DECREF(ptrs);
        Py_DECREF(keep);
        Py_RETURN_NONE;
    }
    PyObject* res = PyTuple_Pack(2, ptrs, keep);
    Py_DECREF(ptrs);
    Py_DECREF(keep);
    return res;
}

PyMethodDef methods[] = {
    {"layout_key", layout_key, METH_O, "checker._layout_key over a record list"},
    {"group_by_id", group_by_id, METH_O, "Trace.by_id positions + merge_view structure keys"},
    {"host_bytes", host_bytes, METH_O, "checker._host_bytes over a record list (None: not torch payloads)"},
    {"resident_ptrs", resident_ptrs, METH_VARARGS, "device._resolve_resident's fast case"},
    {nullptr, nullptr, 0, nullptr},
};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_td_host", "warm-check record walks", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__td_host() {
    s_payload = PyUnicode_InternFromString("payload");
    s_id = PyUnicode_InternFromString("id");
    s_encode = PyUnicode_InternFromString("encode");
    s_rank_meta = PyUnicode_InternFromString("rank_meta");
    s_as_tuple = PyUnicode_InternFromString("as_tuple");
    s_mapping = PyUnicode_InternFromString("mapping");
    s_sig_id = PyUnicode_InternFromString("sig_id");
    s_replica = PyUnicode_InternFromString("replica_group_size");
    s_dtype_code = PyUnicode_InternFromString("dtype_code");
    s_text = PyUnicode_InternFromString("_text");
    s_t = PyUnicode_InternFromString("_t");
    return PyModule_Create(&module);
}
