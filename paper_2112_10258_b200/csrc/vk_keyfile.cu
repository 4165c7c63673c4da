// vk_keyfile.cu -- host-side (CPU) formatter for the reference's keypoint /
// descriptor text files (keyfiles.py:35-122): one line per record,
//   x y z sigma octave level dog_value sign [r00 .. r22] [payload]
// with every real as "%.9g" (correctly rounded by both CPython and glibc,
// so the bytes match the reference writer), payload = ranks as decimal ints
// or packed bits as lowercase hex.  Writes straight from the
// structure-of-arrays the device pipeline returns, no per-record objects.
#include <stdio.h>
#include <string.h>

#include "vk_common.cuh"

extern "C" long long vk_format_records(long long n, const double* pos, const double* sigma, const int* octave,
                                       const int* level, const double* dog, const signed char* sign,
                                       const double* rot, const unsigned char* payload, int payload_kind,
                                       int payload_len, char* out, long long cap) {
    if (n < 0 || (n > 0 && (!pos || !sigma || !octave || !level || !dog || !sign)) || payload_kind < 0 ||
        payload_kind > 2 || (payload_kind && (!payload || payload_len < 1)) || cap < 0) {
        vk::set_error("vk_format_records: bad arguments");
        return -1;
    }
    static const char* hex = "0123456789abcdef";
    long long w = 0;
    char line[4096];
    for (long long i = 0; i < n; ++i) {
        int k = snprintf(line, sizeof(line), "%.9g %.9g %.9g %.9g %d %d %.9g %s", pos[3 * i], pos[3 * i + 1],
                         pos[3 * i + 2], sigma[i], octave[i], level[i], dog[i], sign[i] > 0 ? "peak" : "valley");
        if (rot)
            for (int e = 0; e < 9; ++e) k += snprintf(line + k, sizeof(line) - k, " %.9g", rot[9 * i + e]);
        if (payload_kind == 1) {  // ranks, one byte each
            for (int e = 0; e < payload_len && k < (int)sizeof(line) - 8; ++e)
                k += snprintf(line + k, sizeof(line) - k, " %d", (int)payload[(long long)payload_len * i + e]);
        } else if (payload_kind == 2) {  // packed bits -> hex
            line[k++] = ' ';
            for (int e = 0; e < payload_len && k < (int)sizeof(line) - 4; ++e) {
                const unsigned char b = payload[(long long)payload_len * i + e];
                line[k++] = hex[b >> 4];
                line[k++] = hex[b & 15];
            }
        }
        line[k++] = '\n';
        if (w + k <= cap) memcpy(out + w, line, k);
        w += k;
    }
    return w;  // bytes needed; the caller retries with a larger buffer if w > cap
}
