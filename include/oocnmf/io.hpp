// Forwarder: the reference header name (include/oocnmf/io.hpp) resolves to the B200 host core.
#pragma once
#include "oocnmf_b200/oocnmf.hpp"
