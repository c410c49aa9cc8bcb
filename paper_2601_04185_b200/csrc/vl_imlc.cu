// IMLC correspondence-field header parser (host code).
//
// Reference: matchio.read_field (matchio.py:158-200) and the layout in the
// module docstring (:9-20).  The checks run in the reference's order — each
// `take` can fail as truncated, then magic, version, and trailing bytes — and
// report the same byte offsets, so the Python wrapper raises the same
// FieldFormatError subclass with the same message.  Record content is not
// touched here: the lift kernels read the records in place and validate them
// on the GPU (vl_lift.cu).
#include <cstring>
#include "visloc_b200.h"

namespace {

struct Reader {
  const uint8_t* p;
  int64_t len, off;
  vl_imlc_header* h;
  // matchio.read_field.take: a short read is FieldTruncatedError at `off`
  bool take(int64_t n, const char* what) {
    if (off + n > len) {
      h->status = VL_IMLC_TRUNCATED;
      h->error_offset = off;
      h->need = n;
      h->have = len - off;
      h->what = what;
      return false;
    }
    off += n;
    return true;
  }
  uint32_t u32(int64_t at) const {
    uint32_t v;
    std::memcpy(&v, p + at, 4);  // little-endian host (x86-64 / aarch64)
    return v;
  }
  double f64(int64_t at) const {
    double v;
    std::memcpy(&v, p + at, 8);
    return v;
  }
};

}  // namespace

extern "C" int vl_imlc_parse(const uint8_t* blob, int64_t len, vl_imlc_header* out) {
  if (!out || len < 0 || (len > 0 && !blob)) return VL_ERR_INVALID;
  std::memset(out, 0, sizeof(*out));
  Reader r{blob, len, 0, out};
  if (!r.take(4, "magic")) return VL_OK;
  std::memcpy(out->magic, blob, 4);
  if (std::memcmp(blob, "IMLC", 4) != 0) {
    out->status = VL_IMLC_MAGIC;
    out->error_offset = 0;
    return VL_OK;
  }
  if (!r.take(4, "version")) return VL_OK;
  out->version = r.u32(4);
  if (out->version != 1) {
    out->status = VL_IMLC_VERSION;
    out->error_offset = 4;
    return VL_OK;
  }
  if (!r.take(4, "source id length")) return VL_OK;
  out->source_len = r.u32(r.off - 4);
  out->source_off = r.off;
  if (!r.take(out->source_len, "source id")) return VL_OK;
  if (!r.take(4, "target id length")) return VL_OK;
  out->target_len = r.u32(r.off - 4);
  out->target_off = r.off;
  if (!r.take(out->target_len, "target id")) return VL_OK;
  if (!r.take(8, "grid dimensions")) return VL_OK;
  out->grid_w = r.u32(r.off - 8);
  out->grid_h = r.u32(r.off - 4);
  if (!r.take(16, "scale factors")) return VL_OK;
  out->scale_x = r.f64(r.off - 16);
  out->scale_y = r.f64(r.off - 8);
  out->records_off = r.off;
  const uint64_t nrec = (uint64_t)out->grid_w * (uint64_t)out->grid_h;
  if (nrec > (uint64_t)(len / 12)) {  // cannot fit (also guards 12 * nrec overflow)
    out->status = VL_IMLC_TRUNCATED;
    out->error_offset = r.off;
    out->need = nrec <= (uint64_t)(INT64_MAX / 12) ? (int64_t)(12 * nrec) : -1;  // -1: caller recomputes
    out->have = len - r.off;
    out->what = "records";
    return VL_OK;
  }
  if (!r.take(12 * (int64_t)nrec, "records")) return VL_OK;
  if (r.off != len) {
    out->status = VL_IMLC_TRAILING;
    out->error_offset = r.off;
    out->have = len - r.off;
    return VL_OK;
  }
  out->status = VL_IMLC_OK;
  return VL_OK;
}
