/* pack.c -- Trace records -> SoA columns in one pass (CPython extension `_pack`).
 *
 * Host-side ingest for the drop-in API (compute_report(Trace), metrics.py:125-154):
 * the reference keeps records as Python objects (model.py:51-71); the engine needs
 * packed start / end / dense-id / kind columns.  The pure-Python packer
 * (packing._pack_side) walks the records five times with interpreted attribute
 * lookups and hashes enum members (Enum.__hash__ runs Python code); this walks them
 * once with interned attribute names and maps the state / kind member to its code by
 * IDENTITY (members are singletons).
 *
 * pack_side(records, res_attr, kind_attr, dense, members, start, end, res, kind) -> bool
 *   records   sequence of HostRecord / DeviceRecord
 *   res_attr  "rank" / "device_id";  kind_attr  "state" / "kind"
 *   dense     dict id -> dense index
 *   members   tuple of enum members, position = code
 *   start, end (u64), res (i32), kind (u8): writable buffers of len(records)
 * Returns False (columns unspecified) as soon as a record is not a plain in-range
 * int timestamp pair or has an unknown member / id: the caller then runs the exact
 * Python path, which produces the reference's quarantine messages.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

static PyObject *s_interval, *s_start, *s_end;

static int u64_of(PyObject *v, unsigned long long *out)
{
    if (!PyLong_CheckExact(v)) return 0;   /* bool / float / int subclasses: exact path */
    unsigned long long x = PyLong_AsUnsignedLongLong(v);
    if (x == (unsigned long long)-1 && PyErr_Occurred()) {
        PyErr_Clear();                     /* negative or beyond 64 bits */
        return 0;
    }
    *out = x;
    return 1;
}

static PyObject *pack_side(PyObject *self, PyObject *args)
{
    PyObject *seq, *res_attr, *kind_attr, *dense, *members;
    Py_buffer bs, be, br, bk;
    (void)self;
    if (!PyArg_ParseTuple(args, "OUUO!O!w*w*w*w*", &seq, &res_attr, &kind_attr, &PyDict_Type, &dense, &PyTuple_Type,
                          &members, &bs, &be, &br, &bk))
        return NULL;
    PyObject *fast = PySequence_Fast(seq, "records must be a sequence");
    int ok = 0;
    if (!fast) goto done;
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
    if (bs.len < n * 8 || be.len < n * 8 || br.len < n * 4 || bk.len < n) {
        PyErr_SetString(PyExc_ValueError, "output buffers too small");
        Py_DECREF(fast);
        goto done;
    }
    PyObject **items = PySequence_Fast_ITEMS(fast);
    const Py_ssize_t nm = PyTuple_GET_SIZE(members);
    uint64_t *S = (uint64_t *)bs.buf, *E = (uint64_t *)be.buf;
    int32_t *R = (int32_t *)br.buf;
    uint8_t *K = (uint8_t *)bk.buf;
    ok = 1;
    for (Py_ssize_t i = 0; i < n && ok; ++i) {
        PyObject *rec = items[i];
        PyObject *iv = PyObject_GetAttr(rec, s_interval);
        if (!iv) { ok = -1; break; }
        PyObject *s = PyObject_GetAttr(iv, s_start), *e = s ? PyObject_GetAttr(iv, s_end) : NULL;
        Py_DECREF(iv);
        if (!s || !e) { Py_XDECREF(s); ok = -1; break; }
        unsigned long long sv = 0, ev = 0;
        ok = u64_of(s, &sv) && u64_of(e, &ev);
        Py_DECREF(s);
        Py_DECREF(e);
        if (!ok) break;
        S[i] = sv;
        E[i] = ev;
        PyObject *r = PyObject_GetAttr(rec, res_attr);
        if (!r) { ok = -1; break; }
        PyObject *d = PyDict_GetItemWithError(dense, r);   /* borrowed */
        Py_DECREF(r);
        if (!d) { if (PyErr_Occurred()) ok = -1; else ok = 0; break; }
        const long dv = PyLong_AsLong(d);
        if (dv == -1 && PyErr_Occurred()) { ok = -1; break; }
        R[i] = (int32_t)dv;
        PyObject *k = PyObject_GetAttr(rec, kind_attr);
        if (!k) { ok = -1; break; }
        Py_ssize_t code = -1;
        for (Py_ssize_t j = 0; j < nm; ++j)
            if (PyTuple_GET_ITEM(members, j) == k) { code = j; break; }
        Py_DECREF(k);
        if (code < 0) { ok = 0; break; }
        K[i] = (uint8_t)code;
    }
    Py_DECREF(fast);
done:
    PyBuffer_Release(&bs);
    PyBuffer_Release(&be);
    PyBuffer_Release(&br);
    PyBuffer_Release(&bk);
    if (ok < 0 || PyErr_Occurred()) return NULL;
    return PyBool_FromLong(ok);
}

/* is_canonical(records, res_attr, kind_attr, members_by_value, stream_attr_or_None) -> bool
 * True iff the records are already in the canonical order of Trace.__post_init__
 * (model.py: _canonical_host / _canonical_device keys, the reference's model.py:74-80):
 * (res, start, end, member rank by .value[, stream with None -> -1]) non-decreasing.
 * members_by_value lists the enum members in ascending .value order.  Anything the
 * check cannot decide in 64-bit integers returns False and the caller sorts. */
static int key_of(PyObject *rec, PyObject *res_attr, PyObject *kind_attr, PyObject *members, PyObject *stream_attr,
                  long long key[5])
{
    PyObject *r = PyObject_GetAttr(rec, res_attr);
    if (!r) return -1;
    int ok = PyLong_CheckExact(r);
    key[0] = ok ? PyLong_AsLongLong(r) : 0;
    Py_DECREF(r);
    if (!ok || (key[0] == -1 && PyErr_Occurred())) { PyErr_Clear(); return 0; }
    PyObject *iv = PyObject_GetAttr(rec, s_interval);
    if (!iv) return -1;
    PyObject *s = PyObject_GetAttr(iv, s_start), *e = s ? PyObject_GetAttr(iv, s_end) : NULL;
    Py_DECREF(iv);
    if (!s || !e) { Py_XDECREF(s); return -1; }
    unsigned long long sv = 0, ev = 0;
    ok = u64_of(s, &sv) && u64_of(e, &ev);
    Py_DECREF(s);
    Py_DECREF(e);
    if (!ok) return 0;
    key[1] = (long long)(sv ^ 0x8000000000000000ull);   /* order-preserving for signed compare */
    key[2] = (long long)(ev ^ 0x8000000000000000ull);
    PyObject *k = PyObject_GetAttr(rec, kind_attr);
    if (!k) return -1;
    key[3] = -1;
    for (Py_ssize_t j = 0; j < PyTuple_GET_SIZE(members); ++j)
        if (PyTuple_GET_ITEM(members, j) == k) { key[3] = j; break; }
    Py_DECREF(k);
    if (key[3] < 0) return 0;
    key[4] = 0;
    if (stream_attr != Py_None) {
        PyObject *st = PyObject_GetAttr(rec, stream_attr);
        if (!st) return -1;
        if (st == Py_None) key[4] = -1;
        else if (PyLong_CheckExact(st)) {
            key[4] = PyLong_AsLongLong(st);
            if (key[4] == -1 && PyErr_Occurred()) { PyErr_Clear(); Py_DECREF(st); return 0; }
        } else { Py_DECREF(st); return 0; }
        Py_DECREF(st);
    }
    return 1;
}

static PyObject *is_canonical(PyObject *self, PyObject *args)
{
    PyObject *seq, *res_attr, *kind_attr, *members, *stream_attr;
    (void)self;
    if (!PyArg_ParseTuple(args, "OUUO!O", &seq, &res_attr, &kind_attr, &PyTuple_Type, &members, &stream_attr))
        return NULL;
    PyObject *fast = PySequence_Fast(seq, "records must be a sequence");
    if (!fast) return NULL;
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
    PyObject **items = PySequence_Fast_ITEMS(fast);
    long long prev[5], cur[5];
    int ok = 1;
    for (Py_ssize_t i = 0; i < n && ok == 1; ++i) {
        ok = key_of(items[i], res_attr, kind_attr, members, stream_attr, cur);
        if (ok != 1) break;
        if (i > 0) {
            int c = 0;
            for (int f = 0; f < 5 && c == 0; ++f) c = (prev[f] > cur[f]) - (prev[f] < cur[f]);
            if (c > 0) ok = 0;
        }
        for (int f = 0; f < 5; ++f) prev[f] = cur[f];
    }
    Py_DECREF(fast);
    if (ok < 0) return NULL;
    return PyBool_FromLong(ok == 1);
}

/* make_records(rec_cls, iv_cls, res_name, kind_name, members, res, kinds, starts, ends,
 *              stream_name, streams) -> list
 * Native columns (read_trace / import_mapped) -> record objects, exactly what the frozen
 * dataclasses' generated __init__ does (object.__new__ + object.__setattr__ per field),
 * without running Python bytecode per record.  res int64, kinds u8 (code -> members[code]),
 * starts / ends u64, streams int64 (< 0 -> None) or None when the class has no stream. */
static PyObject *s_e_start, *s_e_end;

static PyObject *new_obj(PyObject *cls)
{
    static PyObject *empty = NULL;
    if (!empty && !(empty = PyTuple_New(0))) return NULL;
    return PyBaseObject_Type.tp_new((PyTypeObject *)cls, empty, NULL);
}

static PyObject *make_records(PyObject *self, PyObject *args)
{
    PyObject *rec_cls, *iv_cls, *res_name, *kind_name, *members, *stream_name, *streams_obj;
    Py_buffer br, bk, bs, be, bt;
    (void)self;
    if (!PyArg_ParseTuple(args, "OOUUO!y*y*y*y*OO", &rec_cls, &iv_cls, &res_name, &kind_name, &PyTuple_Type, &members,
                          &br, &bk, &bs, &be, &stream_name, &streams_obj))
        return NULL;
    PyObject *out = NULL;
    int have_streams = streams_obj != Py_None;
    bt.buf = NULL;
    if (have_streams && PyObject_GetBuffer(streams_obj, &bt, PyBUF_SIMPLE) < 0) goto done;
    const Py_ssize_t n = bs.len / 8;
    if (br.len < n * 8 || bk.len < n || be.len < n * 8 || (have_streams && bt.len < n * 8)) {
        PyErr_SetString(PyExc_ValueError, "column lengths disagree");
        goto done;
    }
    const int64_t *R = (const int64_t *)br.buf, *T = have_streams ? (const int64_t *)bt.buf : NULL;
    const uint8_t *K = (const uint8_t *)bk.buf;
    const uint64_t *S = (const uint64_t *)bs.buf, *E = (const uint64_t *)be.buf;
    const Py_ssize_t nm = PyTuple_GET_SIZE(members);
    out = PyList_New(n);
    if (!out) goto done;
    for (Py_ssize_t i = 0; i < n; ++i) {
        if (K[i] >= nm) { PyErr_SetString(PyExc_ValueError, "kind code out of range"); goto fail; }
        PyObject *iv = new_obj(iv_cls);
        if (!iv) goto fail;
        PyObject *a = PyLong_FromUnsignedLongLong(S[i]), *b = PyLong_FromUnsignedLongLong(E[i]);
        int bad = !a || !b || PyObject_GenericSetAttr(iv, s_e_start, a) < 0 || PyObject_GenericSetAttr(iv, s_e_end, b) < 0;
        Py_XDECREF(a);
        Py_XDECREF(b);
        if (bad) { Py_DECREF(iv); goto fail; }
        PyObject *rec = new_obj(rec_cls);
        if (!rec) { Py_DECREF(iv); goto fail; }
        PyObject *r = PyLong_FromLongLong(R[i]);
        bad = !r || PyObject_GenericSetAttr(rec, res_name, r) < 0 ||
              PyObject_GenericSetAttr(rec, kind_name, PyTuple_GET_ITEM(members, K[i])) < 0 ||
              PyObject_GenericSetAttr(rec, s_interval, iv) < 0;
        Py_XDECREF(r);
        Py_DECREF(iv);
        if (!bad && stream_name != Py_None) {
            PyObject *st = (T && T[i] >= 0) ? PyLong_FromLongLong(T[i]) : (Py_INCREF(Py_None), Py_None);
            bad = !st || PyObject_GenericSetAttr(rec, stream_name, st) < 0;
            Py_XDECREF(st);
        }
        if (bad) { Py_DECREF(rec); goto fail; }
        PyList_SET_ITEM(out, i, rec);   /* steals */
    }
    goto done;
fail:
    Py_CLEAR(out);
done:
    PyBuffer_Release(&br);
    PyBuffer_Release(&bk);
    PyBuffer_Release(&bs);
    PyBuffer_Release(&be);
    if (bt.buf) PyBuffer_Release(&bt);
    return out;
}

/* sort_keys(records, res_attr, kind_attr, members_by_value, stream_attr_or_None,
 *           res_out i64, start_out u64, end_out u64, kind_out u8, stream_out i64) -> bool
 * The canonical-order key columns of every record (key_of above), for a stable numpy
 * lexsort; False when some key is not decidable in 64-bit integers (the caller sorts
 * with the key function instead). */
static PyObject *sort_keys(PyObject *self, PyObject *args)
{
    PyObject *seq, *res_attr, *kind_attr, *members, *stream_attr;
    Py_buffer br, bs, be, bk, bt;
    (void)self;
    if (!PyArg_ParseTuple(args, "OUUO!Ow*w*w*w*w*", &seq, &res_attr, &kind_attr, &PyTuple_Type, &members, &stream_attr,
                          &br, &bs, &be, &bk, &bt))
        return NULL;
    PyObject *fast = PySequence_Fast(seq, "records must be a sequence");
    int ok = 0;
    if (fast) {
        const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
        PyObject **items = PySequence_Fast_ITEMS(fast);
        if (br.len < n * 8 || bs.len < n * 8 || be.len < n * 8 || bk.len < n || bt.len < n * 8) {
            PyErr_SetString(PyExc_ValueError, "output buffers too small");
        } else {
            int64_t *R = (int64_t *)br.buf, *T = (int64_t *)bt.buf;
            uint64_t *S = (uint64_t *)bs.buf, *E = (uint64_t *)be.buf;
            uint8_t *K = (uint8_t *)bk.buf;
            long long key[5];
            ok = 1;
            for (Py_ssize_t i = 0; i < n && ok == 1; ++i) {
                ok = key_of(items[i], res_attr, kind_attr, members, stream_attr, key);
                if (ok != 1) break;
                R[i] = key[0];
                S[i] = (uint64_t)key[1] ^ 0x8000000000000000ull;
                E[i] = (uint64_t)key[2] ^ 0x8000000000000000ull;
                K[i] = (uint8_t)key[3];
                T[i] = key[4];
            }
        }
        Py_DECREF(fast);
    }
    PyBuffer_Release(&br);
    PyBuffer_Release(&bs);
    PyBuffer_Release(&be);
    PyBuffer_Release(&bk);
    PyBuffer_Release(&bt);
    if (ok < 0 || PyErr_Occurred()) return NULL;
    return PyBool_FromLong(ok == 1);
}

static PyMethodDef methods[] = {
    {"sort_keys", sort_keys, METH_VARARGS, "canonical-order key columns (64-bit decidable?)"},
    {"make_records", make_records, METH_VARARGS, "native columns -> record objects (the dataclasses' own __init__ effect)"},
    {"pack_side", pack_side, METH_VARARGS, "records -> (start, end, dense id, kind) columns; False: use the exact path"},
    {"is_canonical", is_canonical, METH_VARARGS, "records already in canonical Trace order (64-bit decidable)?"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pack", NULL, -1, methods};

PyMODINIT_FUNC PyInit__pack(void)
{
    s_interval = PyUnicode_InternFromString("interval");
    s_start = PyUnicode_InternFromString("start");
    s_end = PyUnicode_InternFromString("end");
    s_e_start = s_start;
    s_e_end = s_end;
    if (!s_interval || !s_start || !s_end) return NULL;
    return PyModule_Create(&module);
}
