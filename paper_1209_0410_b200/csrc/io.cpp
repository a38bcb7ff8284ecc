// io.cpp -- bvecs / fvecs record I/O (the reference's vecio module,
// proj/src/vecio.cpp:18-85; layout SPEC.md:129): every record is a
// little-endian u32 dimension followed by `dim` payload entries (u8 for
// bvecs, f32 for fvecs); the dimension is constant across records.
//
// HCG_BVECS / HCG_FVECS exchange u8 rows: fvecs components must be byte
// values of the index view (offset + b * scale), bvecs bytes are the
// reference's widened floats as-is.  HCG_FVECS_F32 exchanges the float
// components themselves (rows = n x dim floats) for HCG_F32 indexes.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hcg.h"

namespace hcg {
hcg_status set_error(hcg_status code, const std::string& msg);
}

namespace {
struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};
}  // namespace

extern "C" {

void hcg_free_buffer(void* p) { std::free(p); }

hcg_status hcg_read_vectors(const char* path, uint32_t format, float offset, float scale, uint8_t** rows_out,
                            uint64_t* n_out, uint32_t* dim_out) {
    using hcg::set_error;
    if (!path || !rows_out || !n_out || !dim_out) return set_error(HCG_EINVAL, "null argument");
    if (format > HCG_FVECS_F32) return set_error(HCG_EINVAL, "unknown vector format");
    const size_t esize = format == HCG_FVECS_F32 ? 4 : 1;
    *rows_out = nullptr;
    *n_out = 0;
    *dim_out = 0;
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f) return set_error(HCG_EIO, std::string("cannot open ") + path);
    std::vector<uint8_t> rows;
    std::vector<float> fbuf;
    uint32_t dim = 0;
    uint64_t n = 0;
    while (true) {
        uint32_t rec = 0;
        const size_t got = std::fread(&rec, 1, 4, fh.f);
        if (got == 0) break;  // clean end of file
        if (got != 4) return set_error(HCG_EIO, std::string(path) + ": truncated record header");
        if (rec == 0) return set_error(HCG_EIO, std::string(path) + ": zero-dimension record");
        if (n == 0) {
            dim = rec;
        } else if (rec != dim) {
            return set_error(HCG_EIO, std::string(path) + ": inconsistent dimension header (" + std::to_string(rec) +
                                          " vs " + std::to_string(dim) + ")");
        }
        const size_t at = rows.size();
        rows.resize(at + size_t(dim) * esize);
        if (format == HCG_FVECS_F32) {
            float* dst = reinterpret_cast<float*>(rows.data() + at);  // vector<uint8_t> storage: memcpy-safe
            fbuf.resize(dim);
            if (std::fread(fbuf.data(), 4, dim, fh.f) != dim)
                return set_error(HCG_EIO, std::string(path) + ": truncated fvecs payload");
            for (uint32_t j = 0; j < dim; ++j)
                if (!std::isfinite(fbuf[j]))
                    return set_error(HCG_EIO, std::string(path) + ": non-finite component in record " + std::to_string(n));
            std::memcpy(dst, fbuf.data(), size_t(dim) * 4);
        } else if (format == HCG_BVECS) {
            if (std::fread(rows.data() + at, 1, dim, fh.f) != dim)
                return set_error(HCG_EIO, std::string(path) + ": truncated bvecs payload");
        } else {
            fbuf.resize(dim);
            if (std::fread(fbuf.data(), 4, dim, fh.f) != dim)
                return set_error(HCG_EIO, std::string(path) + ": truncated fvecs payload");
            for (uint32_t j = 0; j < dim; ++j) {
                const float x = fbuf[j];
                if (!std::isfinite(x))
                    return set_error(HCG_EIO, std::string(path) + ": non-finite component in record " + std::to_string(n));
                const float b = std::nearbyint((x - offset) / scale);
                if (!(b >= 0.0f && b <= 255.0f) || offset + b * scale != x)
                    return set_error(HCG_EINVAL, std::string(path) + ": component of record " + std::to_string(n) +
                                                     " is not a byte value of the index view");
                rows[at + j] = uint8_t(b);
            }
        }
        ++n;
    }
    uint8_t* out = static_cast<uint8_t*>(std::malloc(rows.empty() ? 1 : rows.size()));
    if (!out) return set_error(HCG_ENOMEM, "host allocation failed");
    if (!rows.empty()) std::memcpy(out, rows.data(), rows.size());
    *rows_out = out;
    *n_out = n;
    *dim_out = dim;
    return HCG_OK;
}

hcg_status hcg_write_vectors(const char* path, uint32_t format, float offset, float scale, const uint8_t* rows,
                             uint64_t n, uint32_t dim) {
    using hcg::set_error;
    if (!path || (n && !rows)) return set_error(HCG_EINVAL, "null argument");
    if (format > HCG_FVECS_F32) return set_error(HCG_EINVAL, "unknown vector format");
    if (n && dim == 0) return set_error(HCG_EINVAL, "zero dimension");
    File fh;
    fh.f = std::fopen(path, "wb");
    if (!fh.f) return set_error(HCG_EIO, std::string("cannot open ") + path + " for writing");
    std::vector<float> fbuf(dim);
    for (uint64_t i = 0; i < n; ++i) {
        bool ok = std::fwrite(&dim, 4, 1, fh.f) == 1;
        if (format == HCG_FVECS_F32) {
            ok = ok && std::fwrite(rows + i * dim * 4, 4, dim, fh.f) == dim;
        } else if (format == HCG_BVECS) {
            ok = ok && std::fwrite(rows + i * dim, 1, dim, fh.f) == dim;
        } else {
            for (uint32_t j = 0; j < dim; ++j) fbuf[j] = offset + float(rows[i * dim + j]) * scale;
            ok = ok && std::fwrite(fbuf.data(), 4, dim, fh.f) == dim;
        }
        if (!ok) return set_error(HCG_EIO, std::string("write failed: ") + path);
    }
    return HCG_OK;
}

}  // extern "C"
