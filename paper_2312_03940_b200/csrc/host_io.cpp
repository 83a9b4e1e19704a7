// Host-side PECG graph parsing (format of /root/reference/pkg/src/peakann/vamana.py:229-267):
// the per-vertex records [u32 degree, degree x u32 ids] are variable-length,
// so the record offsets form a chain; one sequential pass resolves them and
// writes the padded (n, R) int32 adjacency and the degrees straight into the
// caller's (pinned) buffers, ready for one upload.
#include <cstdint>
#include <cstring>

#include "../../include/peakann_b200.h"

extern "C" int pk_parse_pecg(const uint32_t* words, int64_t nwords, int64_t n, int64_t R, int32_t* adj,
                             int32_t* deg, int64_t* info) {
    int64_t pos = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (pos >= nwords) {
            info[0] = i;
            return 3;  // truncated at vertex i
        }
        const uint32_t d = words[pos];
        if ((int64_t)d > R) {
            info[0] = i;
            info[1] = d;
            return 4;  // degree above the bound
        }
        if (pos + 1 + (int64_t)d > nwords) {
            info[0] = i;
            return 3;
        }
        int32_t* row = adj + i * R;
        std::memcpy(row, words + pos + 1, sizeof(uint32_t) * d);
        for (int64_t e = d; e < R; ++e) row[e] = -1;
        deg[i] = (int32_t)d;
        pos += 1 + d;
    }
    if (pos != nwords) {
        info[0] = (nwords - pos) * 4;
        return 5;  // trailing bytes
    }
    return 0;
}
