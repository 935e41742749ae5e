// main() of the reference unit tests run on the B200 adapter (see doctest.h)
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
