// The NSW = 2 instantiations of the warp-strip passes (see the note at the top of
// mgb_stream3.cu): the same source, compiled as a second translation unit so that the two
// halves build in parallel.
#define MGB_S3_PART 2
#include "mgb_stream3.cu"
